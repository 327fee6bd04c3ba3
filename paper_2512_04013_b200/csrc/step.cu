// augsched_step kernels (see step.cuh).  sm_100a, compiled with -fmad=false.
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include "step.cuh"
#include "select.cuh"

namespace augsched {

namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef AUGSCHED_SORT_NT
#define AUGSCHED_SORT_NT 256
#endif
#ifndef AUGSCHED_SORT_ITEMS
#define AUGSCHED_SORT_ITEMS 16
#endif
#ifndef AUGSCHED_SORT_BALLOT
#define AUGSCHED_SORT_BALLOT 1
#endif
constexpr int KNT = 256;                      // keys kernel threads
constexpr int SNT = AUGSCHED_SORT_NT;         // sort-pass threads
constexpr int SITEMS = AUGSCHED_SORT_ITEMS;   // items per thread per sort tile
constexpr int STILE = SNT * SITEMS;           // elements per tile
constexpr int SW = SNT / 32;

__device__ __forceinline__ void flag_err(uint32_t* e, uint32_t bits) { atomicOr(e, bits); }

__device__ __forceinline__ long long ld_ll(const long long* p) { return *(volatile const long long*)p; }

// ------------------------------------------------------------------ setup
__global__ void coef_kernel(augsched_config cfg, const augsched_instance_params* ip, Coef* coef,
                            uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) coef[i] = make_coef(cfg, ip[i]);
}

// Claim key of record j of a batch (see StepState::claimA): a later batch
// has a smaller key; within a batch the lower index wins, and in the
// RETURN/NEW/IMPORT phase a RETURN wins over a NEW/IMPORT (the oracle applies
// returns first, B6).
__device__ __forceinline__ unsigned long long claim_key(uint32_t batch, uint32_t prio, uint32_t j) {
  return ((unsigned long long)(0xFFFFFFFFu - batch) << 32) | ((unsigned long long)prio << 31) | j;
}

// convert per-instance ids to global slot indices, validate kinds/ids, and
// claim the record's slot for its phase of the coming batch (records j0 + j)
__global__ void rec_fix_kernel(const uint32_t* kind, uint32_t* id, uint32_t n, uint32_t inst,
                               uint32_t MA, uint32_t* err, unsigned long long* claimA,
                               unsigned long long* claimB, uint32_t batch, uint32_t j0) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t k = kind[j], x = id[j];
  if (k < AUGSCHED_K_NEW || k > AUGSCHED_K_IMPORT || x >= MA) {
    flag_err(err, 1u);
    id[j] = 0xffffffffu;
    return;
  }
  const uint32_t g = inst * MA + x;
  id[j] = g;
  if (k == AUGSCHED_K_CALL || k == AUGSCHED_K_FINISH) atomicMin(&claimA[g], claim_key(batch, 0u, j0 + j));
  else atomicMin(&claimB[g], claim_key(batch, k != AUGSCHED_K_RETURN, j0 + j));
}

struct Rec {
  const uint32_t *kind, *id, *la, *lb, *lc, *flags, *last, *ctx, *kv, *cpu, *pend;
  const float* ta;
};

struct Slots {
  uint32_t* st;
  double* V;
  uint32_t* last;
  int32_t *ctx, *kv, *cpu, *pend;
  long long *A, *P, *Aevt, *Asnap;
  const Coef* coef;
  const augsched_instance_params* ip;
  uint32_t MA;
  uint32_t* wkv;   // sticky: an IMPORT created a KV holder outside running / swapped / Preserve-paused
  const unsigned long long *claimA, *claimB;   // winning record per slot and phase (duplicates: E_STATE)
  uint32_t batch;
  uint32_t* gdirty;   // per instance: grant[] positions [0, gdirty) may be nonzero (the full step clears)
  uint32_t* err;      // device error word (AUGSCHED_DEBUG invariant checks: bit 8)
  // time-invariant keys (ranking 3, one instance): slots whose packed word
  // changes are listed per step epoch (records of epoch e and the grants /
  // evictions of step e-1 are marked e); null otherwise
  uint32_t *dmark, *dlist, *dcnt;
  uint32_t ti_ep;
};

constexpr uint32_t TI_DCAP = 8192;   // changed slots one incremental step merges (else a full sort)

__device__ __forceinline__ void mark_dirty(const Slots& S, uint32_t g, uint32_t ep) {
  if (!S.dmark) return;
  if (!S.dlist) { S.dmark[g] = ep; return; }   // batched handles: marks only, no list
  if (atomicExch(&S.dmark[g], ep) != ep) {
    const uint32_t q = atomicAdd(&S.dcnt[ep & 1], 1u);
    if (q < TI_DCAP) S.dlist[(ep & 1) * TI_DCAP + q] = g;
  }
}

#ifdef AUGSCHED_DEBUG
// §8(c).4 after a step's accounting: sum of grants <= B, ledger non-negative
// (A + P <= cap is the simulator's invariant: step-mode IMPORTs may start a
// handle above its capacity)
__device__ __forceinline__ void debug_check_step(const Slots& S, uint32_t inst, unsigned long long gsum,
                                                 long long B, int64_t cap) {
  (void)cap;
  const long long A = *(volatile long long*)&S.A[inst], P = *(volatile long long*)&S.P[inst];
  if ((long long)gsum > (B > 0 ? B : 0) || A < 0 || P < 0) atomicOr(S.err, 8u);
}
#endif

__device__ __forceinline__ void ledger_add(long long* x, long long d) {
  atomicAdd(reinterpret_cast<unsigned long long*>(x), (unsigned long long)d);
}

// engine events of the previous forward: CALL (issue, S~ by Eq.4-8 with the
// actual context, R13) and FINISH
__global__ void rec_phaseA(Rec r, uint32_t n, Slots S, uint32_t* err) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t k = r.kind[j], g = r.id[j];
  if (g == 0xffffffffu || (k != AUGSCHED_K_CALL && k != AUGSCHED_K_FINISH)) return;
  // a second CALL/FINISH for the same slot in one batch is a state violation
  // (the oracle applies the first and rejects the rest)
  if (S.claimA[g] != claim_key(S.batch, 0u, j)) { flag_err(err, 1u); return; }
  mark_dirty(S, g, S.ti_ep);
  const uint32_t inst = g / S.MA;
  const uint32_t st = S.st[g] & 15;
  if (k == AUGSCHED_K_FINISH) {
    if (st < ST_RUN || st > ST_WAIT) { flag_err(err, 1u); return; }
    if (S.kv[g] != 0) ledger_add(&S.A[inst], -(long long)S.kv[g]);
    S.st[g] = ST_NONE; S.kv[g] = 0; S.ctx[g] = 0; S.cpu[g] = 0; S.pend[g] = 0;
    return;
  }
  const int32_t ctx = S.ctx[g], kv = S.kv[g];
  if (st != ST_RUN || S.cpu[g] != 0 || kv != ctx || S.pend[g] != 0) { flag_err(err, 1u); return; }
  const Coef& c = S.coef[inst];
  const int pol = select_policy(c, (uint64_t)ctx, (double)r.ta[j],
                                (uint64_t)(S.Aevt[inst] - (long long)kv), S.ip[inst].policy_mode);
  ledger_add(&S.A[inst], -(long long)kv);
  if (pol == POL_P) ledger_add(&S.P[inst], kv);
  else if (pol == POL_S) { S.cpu[g] = ctx; S.kv[g] = 0; }
  else S.kv[g] = 0;
  S.st[g] = ST_PAUSED | ((uint32_t)pol << 4);
}

__global__ void snap_kernel(const long long* A, long long* Asnap, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) Asnap[i] = A[i];
}

// RETURN (Stage II + final value, routing), NEW (Stage I), IMPORT (restore)
__global__ void rec_phaseBC(Rec r, uint32_t n, Slots S, uint64_t now, uint32_t* err) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t k = r.kind[j], g = r.id[j];
  if (g == 0xffffffffu || k == AUGSCHED_K_CALL || k == AUGSCHED_K_FINISH) return;
  if (S.claimB[g] != claim_key(S.batch, k != AUGSCHED_K_RETURN, j)) { flag_err(err, 1u); return; }
  mark_dirty(S, g, S.ti_ep);
  const uint32_t inst = g / S.MA;
  const Coef& c = S.coef[inst];
  const uint32_t pm = S.ip[inst].policy_mode;
  const uint64_t Asnap = (uint64_t)S.Asnap[inst];
  const uint32_t stv = S.st[g] & 15;
  const bool flag1 = (r.flags[j] & 1u) != 0;
  if (k == AUGSCHED_K_RETURN) {
    if (stv != ST_PAUSED) { flag_err(err, 1u); return; }
    const int pol = (int)((S.st[g] >> 4) & 3);
    const int32_t kv = S.kv[g];
    S.V[g] = intake_stage2(c, pm, pol, (uint64_t)S.ctx[g], r.la[j], r.lb[j], (double)r.ta[j], flag1, Asnap);
    uint32_t ns;
    if (pol == POL_P) { ns = ST_RUN; ledger_add(&S.P[inst], -(long long)kv); ledger_add(&S.A[inst], kv); }
    else if (pol == POL_S) ns = ST_SWAP;
    else ns = ST_WAIT;
    S.pend[g] = (int32_t)r.la[j];
    S.st[g] = ns | ((uint32_t)pol << 4);
    return;
  }
  if (stv != ST_NONE) { flag_err(err, 1u); return; }
  if (k == AUGSCHED_K_NEW) {
    S.V[g] = intake_stage1(c, pm, r.la[j], r.lb[j], (double)r.ta[j], flag1, Asnap);
    S.st[g] = ST_WAIT | ((uint32_t)POL_D << 4);
    S.ctx[g] = 0; S.kv[g] = 0; S.cpu[g] = 0; S.pend[g] = (int32_t)r.la[j];
    S.last[g] = (uint32_t)now;
    return;
  }
  // IMPORT (a last-scheduled time in the future is a state violation:
  // Eq.26's wait now - last would wrap)
  const uint32_t f = r.flags[j];
  const uint32_t ns = (f >> 4) & 7, pol = (f >> 8) & 3;
  const bool st2 = (f >> 12) & 1;
  if (ns < ST_RUN || ns > ST_PAUSED || pol > 2 || (uint64_t)r.last[j] > now) { flag_err(err, 1u); return; }
  S.V[g] = st2 ? intake_stage2(c, pm, (int)pol, r.la[j], r.lb[j], r.lc[j], (double)r.ta[j], flag1, Asnap)
               : intake_stage1(c, pm, r.la[j], r.lb[j], (double)r.ta[j], flag1, Asnap);
  S.st[g] = ns | (pol << 4);
  S.last[g] = r.last[j];
  S.ctx[g] = (int32_t)r.ctx[j]; S.kv[g] = (int32_t)r.kv[j]; S.cpu[g] = (int32_t)r.cpu[j];
  S.pend[g] = (int32_t)r.pend[j];
  if (r.kv[j] > 0 && !(ns == ST_RUN || ns == ST_SWAP || (ns == ST_PAUSED && pol == POL_P))) atomicOr(S.wkv, 1u);
  // one address per instance: skip the atomic for the (common) KV-free import
  if (r.kv[j] != 0) {
    if (ns == ST_PAUSED && pol == POL_P) ledger_add(&S.P[inst], (long long)r.kv[j]);
    else ledger_add(&S.A[inst], (long long)r.kv[j]);
  }
}

// ------------------------------------------------------------------ keys
struct KeyArgs {
  Slots S;
  augsched_config cfg;
  int64_t cap;
  uint64_t now;
  unsigned long long* k0;
  uint32_t* ghist;
  uint32_t* tcnt;      // [4 * n_inst] queued slots per (instance, tier), zero at entry
  long long* budget;
  int npass;
  PassDesc passes[STEP_MAX_PASS];
  uint32_t N;
};

// Packed sort word of one slot: tier:2 | key:32 | slot:30 (tier 3 = not queued).
constexpr int PK_KEY = 30;
constexpr int PK_TIER = 62;
constexpr uint32_t SLOT_MASK = (1u << 30) - 1;
constexpr uint32_t INVALID_SLOT = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t digit_of(unsigned long long x, const PassDesc& d, uint32_t MA) {
  if (d.src == 0) return (uint32_t)(x >> d.shift) & ((1u << d.bits) - 1u);
  return ((((uint32_t)x & SLOT_MASK) / MA) >> d.shift) & 255u;
}

// Score every slot (a4): key = orderable u32 of fp32(V - alpha*wait) for
// queued slots (tier 0 running, 1 swapped, 2 waiting); empty / paused slots
// get tier 3 and sort behind their instance's queue.  Also the token limit of
// each instance (a3), its queue size and the digit histograms of every sort
// pass (warp-aggregated shared atomics).
constexpr int KCNT = 1024;   // per-block (instance, tier) count table of the keys kernel (4 words per instance)

#ifndef AUGSCHED_KEYS_KU
#define AUGSCHED_KEYS_KU 4
#endif
#ifndef AUGSCHED_KEYS_GRIDMUL
#define AUGSCHED_KEYS_GRIDMUL 4
#endif
constexpr int KU = AUGSCHED_KEYS_KU;   // slots in flight per thread in the keys kernel

// Shared histogram increment for bins that are heavily shared within a warp
// (the top digits of similar scores): the lanes holding lane 0's bin add with
// one atomic, the others individually.  All 32 lanes must call it; d < 0
// means no item.
__device__ __forceinline__ void hist_add(uint32_t* h, int d) {
  const int lane = threadIdx.x & 31;
  const int d0 = __shfl_sync(FULL, d, 0);
  const unsigned same = __ballot_sync(FULL, d == d0 && d >= 0);
  if (lane == 0 && same) atomicAdd(&h[d0], (unsigned)__popc(same));
  if (d >= 0 && !((same >> lane) & 1u)) atomicAdd(&h[d], 1u);
}

__global__ void __launch_bounds__(KNT) keys_kernel(KeyArgs a) {
  __shared__ uint32_t h[STEP_HIST_WORDS];
  __shared__ uint32_t qcnt[KCNT];
  const int tid = threadIdx.x, lane = tid & 31;
  const int hw = a.passes[a.npass - 1].hoff + (1 << a.passes[a.npass - 1].bits);
  for (int b = tid; b < hw; b += KNT) h[b] = 0;
  for (int b = tid; b < KCNT; b += KNT) qcnt[b] = 0;
  __syncthreads();
  const uint32_t MA = a.S.MA;
  const bool single = MA == a.N;
  // contiguous chunk per block: the instances it touches are contiguous, so
  // their queue counts aggregate in shared memory (one global atomic per
  // block and instance instead of one per warp)
  const uint32_t chunk = (a.N + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * chunk;
  const uint32_t c1 = c0 + chunk < a.N ? c0 + chunk : a.N;
  const uint32_t i0 = c0 / MA;
  const bool local_cnt = c1 > c0 && (c1 - 1) / MA - i0 < (uint32_t)KCNT / 4;
  uint32_t myq[3] = {0u, 0u, 0u};   // queued slots per tier seen by this thread (single-instance handles)
  if (single) {
    // one instance: its constants in registers, the three scoring words of
    // KU slots loaded together
    const Coef k = a.S.coef[0];
    const augsched_instance_params ip = a.S.ip[0];
    if (c0 == 0 && c1 > 0)
      a.budget[0] = token_limit(a.cfg, k, ip, a.cap, ld_ll(&a.S.A[0]), ld_ll(&a.S.P[0]));
    for (uint32_t base = c0; base < c1; base += KNT * KU) {
      uint32_t stv[KU], lst[KU];
      double V[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const uint32_t s = base + u * KNT + tid;
        stv[u] = 0u; lst[u] = 0u; V[u] = 0.0;
        if (s < c1) { stv[u] = a.S.st[s] & 15; V[u] = a.S.V[s]; lst[u] = a.S.last[s]; }
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const uint32_t s = base + u * KNT + tid;
        const uint32_t tier = (stv[u] >= ST_RUN && stv[u] <= ST_WAIT) ? stv[u] - ST_RUN : 3u;
        const uint32_t key = tier < 3 ? rank_key(k, ip, V[u], a.now, lst[u], s) : 0u;
        const unsigned long long x = ((unsigned long long)tier << PK_TIER) |
                                     ((unsigned long long)key << PK_KEY) | s;
        if (s < c1) {
          a.k0[s] = x;
          if (tier < 3) ++myq[tier];
        }
        for (int p = 0; p < a.npass; ++p)
          hist_add(h + a.passes[p].hoff, s < c1 ? (int)digit_of(x, a.passes[p], MA) : -1);
      }
    }
  } else
  for (uint32_t base = c0; base < c1; base += KNT * KU) {   // block-uniform trip count
    uint32_t stv[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint32_t s = base + u * KNT + tid;
      stv[u] = s < c1 ? a.S.st[s] & 15 : 0u;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint32_t s = base + u * KNT + tid;
      const bool valid = s < c1;
      uint32_t inst = 0, key = 0;
      const uint32_t tier = (stv[u] >= ST_RUN && stv[u] <= ST_WAIT) ? stv[u] - ST_RUN : 3u;
      if (valid) {
        inst = s / MA;
        if (tier < 3)
          key = rank_key(a.S.coef[inst], a.S.ip[inst], a.S.V[s], a.now, a.S.last[s], s - inst * MA);
        if (s == inst * MA)
          a.budget[inst] = token_limit(a.cfg, a.S.coef[inst], a.S.ip[inst], a.cap,
                                       ld_ll(&a.S.A[inst]), ld_ll(&a.S.P[inst]));
      }
      const unsigned long long x = ((unsigned long long)tier << PK_TIER) |
                                   ((unsigned long long)key << PK_KEY) | s;
      if (valid) a.k0[s] = x;
      // queued count per (instance, tier)
      const bool q = valid && tier < 3;
      {
        const unsigned qm = __ballot_sync(FULL, q);
        if (qm) {
          const unsigned peers = __match_any_sync(FULL, q ? (int)(inst * 4 + tier) : -1) & qm;
          if (q && lane == __ffs(peers) - 1) {
            if (local_cnt) atomicAdd(&qcnt[(inst - i0) * 4 + tier], (unsigned)__popc(peers));
            else atomicAdd(&a.tcnt[inst * 4 + tier], (unsigned)__popc(peers));
          }
        }
      }
      for (int p = 0; p < a.npass; ++p) {
        const int d = valid ? (int)digit_of(x, a.passes[p], MA) : -1;
        hist_add(h + a.passes[p].hoff, d);
      }
    }
  }
  if (single) {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      uint32_t q = myq[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(FULL, q, o);
      if (lane == 0 && q) atomicAdd(&qcnt[t], q);
    }
  }
  __syncthreads();
  for (int b = tid; b < hw; b += KNT)
    if (h[b]) atomicAdd(&a.ghist[b], h[b]);
  if (local_cnt)
    for (uint32_t b = tid; b < 4 * ((c1 - 1) / MA - i0 + 1); b += KNT)
      if (qcnt[b]) atomicAdd(&a.tcnt[4 * i0 + b], qcnt[b]);
}

// ------------------------------------------------------------------ sort pass
struct SortArgs {
  const unsigned long long* kin;
  unsigned long long* kout;
  uint32_t n;
  PassDesc d;
  uint32_t MA;
  const uint32_t* ghist;        // this pass's bins
  unsigned long long* status;   // [tiles][1 << RB] tile aggregates
  unsigned long long* gstatus;  // [groups][1 << RB] group aggregates
  uint32_t G;                   // tiles per group
  unsigned long long epoch;
  uint32_t* tile_ctr;
  int final_;                   // last pass: write order (local slot) and key
  uint32_t* order;
  uint32_t* keyout;
};

// Lanes of the warp holding the same RB-bit digit as this lane (d < 0: the
// lane holds no item and is in no other lane's set).  RB + 1 ballots; the
// __match_any_sync variant is kept for comparison (AUGSCHED_SORT_BALLOT=0).
// All 32 lanes hold an item: RB ballots.
template <int RB>
__device__ __forceinline__ unsigned digit_peers_full(uint32_t d) {
  unsigned m = FULL;
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    const unsigned v = __ballot_sync(FULL, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? v : ~v;
  }
  return m;
}

template <int RB>
__device__ __forceinline__ unsigned digit_peers(int d) {
#if AUGSCHED_SORT_BALLOT
  unsigned m = __ballot_sync(FULL, d >= 0);
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    const bool bit = (d >> b) & 1;
    const unsigned v = __ballot_sync(FULL, bit);
    m &= bit ? v : ~v;
  }
  return m;
#else
  return __match_any_sync(FULL, d);
#endif
}

constexpr int LB_BATCH = 8;     // aggregate words loaded together by one thread

// Spin until every word of a strided run carries this pass's epoch; return
// the sum of their counts (the low 32 bits).
__device__ __forceinline__ uint32_t sum_published(volatile unsigned long long* base, uint32_t count,
                                                  size_t stride, unsigned long long ep) {
  uint32_t total = 0;
  for (uint32_t k0 = 0; k0 < count; k0 += LB_BATCH) {
    unsigned long long w[LB_BATCH];
    bool ok;
    do {
#pragma unroll
      for (int k = 0; k < LB_BATCH; ++k)
        w[k] = k0 + k < count ? base[(size_t)(k0 + k) * stride] : (ep << 34);
      ok = true;
#pragma unroll
      for (int k = 0; k < LB_BATCH; ++k) ok &= (w[k] >> 34) == ep;
    } while (!ok);
#pragma unroll
    for (int k = 0; k < LB_BATCH; ++k) total += k0 + k < count ? (uint32_t)w[k] : 0u;
  }
  return total;
}

// One stable LSD counting-sort pass over a digit of RB bits.  Tile = SNT x
// SITEMS elements; each warp ranks its contiguous segment with
// __match_any_sync and warp-private digit counters, one barrier combines
// warps.  The tile's digit offsets come from a two-level aggregate
// look-back with no serial chain: every tile publishes its digit counts, the
// last tile of each group of G tiles publishes the group's counts, and tile
// t (group g) sums the aggregates of groups < g and of the tiles before it in
// its own group (<= 2*sqrt(tiles) independent loads per digit).  Tile ids are
// handed out in launch order by an atomic counter, so every awaited tile has
// started.
template <int RB>
__global__ void __launch_bounds__(SNT) sort_pass_kernel(SortArgs a) {
  constexpr int NB = 1 << RB;
  constexpr int DPT = NB / SNT > 0 ? NB / SNT : 1;   // digits per thread
  __shared__ uint32_t bin_off[NB];
  __shared__ uint32_t wcnt[SW][NB];
  __shared__ uint32_t tbase[NB];
  __shared__ uint32_t wtot[SW];
  __shared__ uint32_t tile_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) tile_s = atomicAdd(a.tile_ctr, 1u);
  for (int w = 0; w < SW; ++w)
    for (int b = tid; b < NB; b += SNT) wcnt[w][b] = 0;
  // exclusive scan of the global digit histogram: thread tid owns bins
  // [tid*DPT, tid*DPT + DPT)
  {
    uint32_t loc[DPT], sum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int b = tid * DPT + j;
      loc[j] = b < NB ? a.ghist[b] : 0u;
      sum += loc[j];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    uint32_t run = inc - sum;
    for (int w = 0; w < warp; ++w) run += wtot[w];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int b = tid * DPT + j;
      if (b < NB) bin_off[b] = run;
      run += loc[j];
    }
  }
  const uint32_t tile = tile_s;
  const size_t seg = (size_t)tile * STILE + (size_t)warp * (32 * SITEMS);
  unsigned long long kk[SITEMS];
  uint32_t rk[SITEMS];
  int dg[SITEMS];
#pragma unroll
  for (int r = 0; r < SITEMS; ++r) {
    const size_t idx = seg + (size_t)r * 32 + lane;
    if (idx < a.n) {
      kk[r] = a.kin[idx];
      dg[r] = (int)digit_of(kk[r], a.d, a.MA);
    } else {
      kk[r] = 0; dg[r] = -1;
    }
  }
  __syncthreads();  // wcnt cleared, bin_off ready
  const unsigned lt = (1u << lane) - 1;
#pragma unroll
  for (int r = 0; r < SITEMS; ++r) {
    const unsigned peers = digit_peers<RB>(dg[r]);
    if (dg[r] >= 0) rk[r] = wcnt[warp][dg[r]] + __popc(peers & lt);
    __syncwarp();
    if (dg[r] >= 0 && lane == __ffs(peers) - 1) wcnt[warp][dg[r]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets of the warps, tile count, decoupled look-back
  volatile unsigned long long* st = a.status;
  volatile unsigned long long* gst = a.gstatus;
  const unsigned long long ep = a.epoch;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = tid * DPT + j;
    if (d >= NB) break;
    uint32_t cnt = 0;
    for (int w = 0; w < SW; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = cnt;
      cnt += c;
    }
    // aggregate word: epoch << 34 | count
    st[(size_t)tile * NB + d] = (ep << 34) | cnt;
    const uint32_t g = tile / a.G, t0 = g * a.G;
    if (tile == t0 + a.G - 1 || tile == gridDim.x - 1)   // last tile of its group
      gst[(size_t)g * NB + d] = (ep << 34) | (sum_published(st + (size_t)t0 * NB + d, tile - t0, NB, ep) + cnt);
    const uint32_t excl = sum_published(gst + d, g, NB, ep) +
                          sum_published(st + (size_t)t0 * NB + d, tile - t0, NB, ep);
    tbase[d] = excl;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SITEMS; ++r) {
    if (dg[r] < 0) continue;
    const uint32_t d = (uint32_t)dg[r];
    const uint32_t pos = bin_off[d] + tbase[d] + wcnt[warp][d] + rk[r];
    if (a.final_) {
      const uint32_t gsl = (uint32_t)kk[r] & SLOT_MASK;
      a.order[pos] = gsl - (gsl / a.MA) * a.MA;
      a.keyout[pos] = (uint32_t)(kk[r] >> PK_KEY);
    } else {
      a.kout[pos] = kk[r];
    }
  }
}

// ------------------------------------------------------------------ block scan helpers
template <int NT>
__device__ __forceinline__ unsigned long long block_incl_scan_u64(unsigned long long x,
                                                                  unsigned long long* wsum,
                                                                  unsigned long long* total) {
  // warp scans, then warp 0 scans the warp totals (wsum holds NT/32 + 1 words:
  // exclusive warp offsets and the block total)
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long t = lane < NW ? wsum[lane] : 0ull;
    unsigned long long c = t;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, c, o);
      if (lane >= o) c += y;
    }
    if (lane < NW) wsum[lane] = c - t;
    if (lane == NW - 1) wsum[NW] = c;
  }
  __syncthreads();
  const unsigned long long base = wsum[warp];
  *total = wsum[NW];
  __syncthreads();
  return base + inc;
}

__device__ __forceinline__ uint32_t slot_demand(const Slots& S, uint32_t g, uint32_t s_in) {
  return demand_of(S.ctx[g], S.kv[g], S.cpu[g], S.pend[g], s_in);
}

constexpr int ANT = 512;    // threads of the per-instance admission kernel
constexpr int ANW = ANT / 32;

// One block per instance, after the sort:
//   a6  grants of the admitted prefix (P_{j-1} < B, partial last, R17)
//   a7  (rare) demote Preserve-paused KV (kv desc, slot asc), then evict from
//       the tail of the order over entries with kv + g > 0, until the grants
//       fit the free KV memory (R20)
//   S9  last = now and the granted batch's token accounting (decode adds one
//       token; the engine reports segment ends with CALL / FINISH records)
//   out  n_active and the per-tier segment starts (from the keys kernel's
//        per-tier counts); grant[j] = 0 for j >= the admitted prefix (the
//        previous step's grants beyond it are cleared)
__global__ void __launch_bounds__(ANT) admit_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                    const long long* budget, const uint32_t* tcnt,
                                                    uint32_t* n_active, uint32_t* tier_off,
                                                    const uint32_t* order, uint32_t* grant,
                                                    uint32_t* admitted) {
  __shared__ unsigned long long wsum[ANW + 1];
  __shared__ SelShm sel;
  __shared__ unsigned long long freed;
  const uint32_t i = blockIdx.x;
  const int tid = threadIdx.x;
  const uint32_t MA = S.MA;
  const size_t base = (size_t)i * MA;
  const long long B = budget[i];
  const uint32_t c0 = tcnt[4 * i], c1 = tcnt[4 * i + 1], c2 = tcnt[4 * i + 2];
  const uint32_t n = c0 + c1 + c2;
  const uint32_t prev_adm = S.gdirty[i];   // earlier steps' grants live in [0, prev_adm)
  // ---- a6 admission
  unsigned long long Prun = 0, gsum = 0;
  uint32_t adm = 0;
  for (uint32_t j0 = 0; j0 < n && (long long)Prun < B; j0 += ANT) {
    const uint32_t j = j0 + tid;
    unsigned long long d = 0;
    if (j < n) d = slot_demand(S, (uint32_t)(base + order[base + j]), cfg.s_in);
    unsigned long long tot;
    const unsigned long long inc = block_incl_scan_u64<ANT>(d, wsum, &tot);
    const unsigned long long ex = Prun + inc - d;
    const bool in = j < n && (long long)ex < B;
    if (in) {
      const unsigned long long g = d < (unsigned long long)B - ex ? d : (unsigned long long)B - ex;
      grant[base + j] = (uint32_t)g;
      gsum += g;
    }
    adm += __syncthreads_count(in);
    Prun += tot;
  }
  unsigned long long need;
  block_incl_scan_u64<ANT>(gsum, wsum, &need);
  long long fr = cap - ld_ll(&S.A[i]) - ld_ll(&S.P[i]);
  // ---- a7 resolution (rare)
  if ((long long)need > fr) {
    if (tid == 0) freed = 0;
    auto getp = [&](uint32_t x, uint64_t& key, uint32_t& w) {
      const size_t g = base + x;
      const uint32_t stv = S.st[g];
      const int32_t kv = S.kv[g];
      if ((stv & 15) != ST_PAUSED || ((stv >> 4) & 3) != POL_P || kv <= 0) return false;
      key = ((uint64_t)(0xFFFFFFFFu - (uint32_t)kv) << 24) | x;
      w = (uint32_t)kv;
      return true;
    };
    wselect<ANT>(sel, MA, (uint64_t)((long long)need - fr), 56, getp);
    {
      const bool f0 = sel.r.found != 0;
      const uint64_t k0 = sel.r.k;
      for (uint32_t x = tid; x < MA; x += ANT) {
        uint64_t key;
        uint32_t w;
        if (getp(x, key, w) && (!f0 || key <= k0)) {
          const size_t g = base + x;
          atomicAdd(&freed, (unsigned long long)w);
          S.kv[g] = 0;
          S.st[g] = ST_PAUSED | ((uint32_t)POL_D << 4);
        }
      }
    }
    __syncthreads();
    if (tid == 0) ledger_add(&S.P[i], -(long long)freed);
    fr += (long long)freed;
    if ((long long)need > fr) {
      auto gete = [&](uint32_t j, uint64_t& key, uint32_t& w) {
        const size_t g = base + order[base + j];
        w = (uint32_t)S.kv[g] + (j < adm ? grant[base + j] : 0u);
        key = (uint64_t)(n - 1 - j);
        return w > 0;
      };
      wselect<ANT>(sel, n, (uint64_t)((long long)need - fr), 24, gete);
      const bool f1 = sel.r.found != 0;
      const uint64_t k1 = sel.r.k;
      __syncthreads();
      long long dA = 0;
      for (uint32_t j = tid; j < n; j += ANT) {
        uint64_t key;
        uint32_t w;
        if (gete(j, key, w) && (!f1 || key <= k1)) {
          const size_t g = base + order[base + j];
          dA -= S.kv[g];
          S.kv[g] = 0;
          S.cpu[g] = 0;
          S.st[g] = ST_WAIT | (S.st[g] & 0x30u);
          if (j < adm) grant[base + j] = 0;
        }
      }
      if (dA) ledger_add(&S.A[i], dA);
    }
  }
  __syncthreads();   // grants final, ledger updates visible in the block
  // ---- S9 + token accounting
  unsigned long long dA = 0;
  for (uint32_t j = tid; j < adm; j += ANT) {
    const uint32_t gr = grant[base + j];
    if (gr == 0) continue;
    const size_t g = base + order[base + j];
    int32_t ctx = S.ctx[g], kv = S.kv[g], cpu = S.cpu[g], pend = S.pend[g];
    if (cpu > 0) { cpu -= (int32_t)gr; kv += (int32_t)gr; }
    else if ((ctx - kv) + pend > 0) {
      const int32_t rc = (int32_t)gr < ctx - kv ? (int32_t)gr : ctx - kv;
      kv += rc;
      const int32_t pp = (int32_t)gr - rc;
      pend -= pp; ctx += pp; kv += pp;
    } else { ctx += 1; kv += 1; }
    dA += gr;
    S.ctx[g] = ctx; S.kv[g] = kv; S.cpu[g] = cpu; S.pend[g] = pend;
    S.last[g] = (uint32_t)now;
    S.st[g] = ST_RUN | (S.st[g] & 0x30u);
  }
  // grants beyond the prefix: zero (the previous step wrote [0, prev_adm))
  for (uint32_t j = adm + tid; j < prev_adm && j < MA; j += ANT) grant[base + j] = 0;
  unsigned long long tot;
  block_incl_scan_u64<ANT>(dA, wsum, &tot);
  if (tid == 0) {
    admitted[i] = adm;
    S.gdirty[i] = adm;
    n_active[i] = n;
    tier_off[3 * i] = 0;
    tier_off[3 * i + 1] = c0;
    tier_off[3 * i + 2] = c0 + c1;
    const long long a = ld_ll(&S.A[i]) + (long long)tot;
    S.A[i] = a;
    S.Aevt[i] = a;
#ifdef AUGSCHED_DEBUG
    debug_check_step(S, i, tot, B, cap);
#endif
  }
}


// ====================================================================== prefix step
// augsched_step_prefix: the same decision round, producing the order only
// for the admitted prefix.  Every queued request has demand >= 1, so the
// admitted prefix lies within the first min(B, n) entries of the order
// (target = min(B, n)); it is found by selection instead of a full sort.
//
// Single-instance handle: one cooperative kernel (pf_step_kernel), one CTA
// of 1,024 threads per SM.
//   phase 1  (speculative) one streaming pass over the slots: packed word
//            of every slot (Eq.26 key), queue size, and every word <= theta
//            appended to a candidate list.  theta is the current word of an
//            anchor slot chosen by the previous step a margin beyond its
//            admitted prefix: every unscheduled score falls by the same
//            alpha*T per iteration (Eq.26), so the anchor keeps about the
//            same rank and the list holds about target + margin words.
//            Exact whenever target <= |list| <= PF_SCAP: the target
//            smallest words are then all <= theta.  The last CTA checks
//            that and, if it holds, finishes the step alone.
//   phase 2  (fallback: first step, a random shuffle, records that moved
//            the anchor, ...) packed words to k0 + histogram of the top
//            12-bit digit; the last CTA locates the bucket b* of the
//            target-th word;
//   phase 3  words below b* -> A (< target of them), in b* -> C; the last
//            CTA selects the smallest of C and finishes.
//   finish   bitonic sort of the candidates in shared memory, admission
//            (R17), resolution (R20, exact selections over all slots),
//            grant accounting, and the next anchor.
// Multi-instance handles: pf_multi_kernel (one CTA per instance).

__device__ __forceinline__ uint32_t pf_target(long long B, uint32_t n) {
  if (B <= 0) return 0u;
  return (unsigned long long)B < n ? (uint32_t)B : n;
}

// Packed word of local slot x of an instance (tier 3 = not queued).
__device__ __forceinline__ unsigned long long slot_word(const Coef& k, const augsched_instance_params& ip,
                                                        uint32_t stv, double V, uint32_t last, uint64_t now,
                                                        uint32_t x) {
  stv &= 15;
  const uint32_t tier = (stv >= ST_RUN && stv <= ST_WAIT) ? stv - ST_RUN : 3u;
  const uint32_t key = tier < 3 ? rank_key(k, ip, V, now, last, x) : 0u;
  return ((unsigned long long)tier << PK_TIER) | ((unsigned long long)key << PK_KEY) | x;
}

#ifdef AUGSCHED_PF_TIMING
// phase timestamps of the prefix-step kernel (profiling builds only)
__device__ unsigned long long g_pf_t[8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PF_T(i, first) do { if (threadIdx.x == 0) { if (first) atomicMin(&g_pf_t[i], gtime()); else atomicMax(&g_pf_t[i], gtime()); } } while (0)
#else
#define PF_T(i, first) do {} while (0)
#endif

constexpr int PNT = 1024;

// The admitted prefix of instance `inst` from `mt` candidate words in sbuf
// (which hold its first `target` order entries): bitonic sort, admission
// (R17), resolution by exact selections over the instance's slots (R20),
// grant accounting.  `keys` are the instance's packed words (local slot in
// the low bits; tier 3 = not queued); `xch` is a second buffer of the same
// size as sbuf for the sort's shared-memory exchanges.
__device__ __forceinline__ void bar_named(uint32_t nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Bitonic sort of 2^LOGP words, one per thread (threads 0 .. 2^LOGP - 1),
// the network fully unrolled: partner distances below 32 by warp shuffles,
// the others through a double-buffered shared exchange.
template <int LOGP>
__device__ __forceinline__ unsigned long long bitonic1(unsigned long long v, unsigned long long* b0,
                                                       unsigned long long* b1) {
  constexpr uint32_t P = 1u << LOGP;
  const uint32_t t = threadIdx.x;
  int xp = 0;
#pragma unroll
  for (int lk = 1; lk <= LOGP; ++lk) {
#pragma unroll
    for (int lj = lk - 1; lj >= 0; --lj) {
      const uint32_t k = 1u << lk, j = 1u << lj;
      unsigned long long pv;
      if (j < 32) {
        pv = __shfl_xor_sync(FULL, v, j);
      } else {
        unsigned long long* xb = xp ? b1 : b0;
        xp ^= 1;
        xb[t] = v;
        bar_named(P);
        pv = xb[t ^ j];
      }
      const bool keep_min = ((t & j) == 0) == ((t & k) == 0);
      const bool lt = pv < v;
      v = (keep_min == lt) ? pv : v;
    }
  }
  return v;
}

// Bitonic sort of 2^LOGP words, E per thread over T = 2^LOGP / E threads
// (index t + e * T), the network fully unrolled: distances >= T inside the
// thread, below 32 by warp shuffles, in between through a double-buffered
// shared exchange (one named barrier over the T threads per stage).
template <int LOGP, int E>
__device__ __forceinline__ void bitonicE(unsigned long long (&v)[E], unsigned long long* b0,
                                         unsigned long long* b1) {
  constexpr uint32_t P = 1u << LOGP, T = P / E;
  static_assert(T >= 32 && T * E == P, "one warp at least");
  const uint32_t t = threadIdx.x;
  int xp = 0;
#pragma unroll
  for (int lk = 1; lk <= LOGP; ++lk) {
#pragma unroll
    for (int lj = lk - 1; lj >= 0; --lj) {
      const uint32_t k = 1u << lk, j = 1u << lj;
      if (j >= T) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int e2 = e ^ (int)(j / T);
          if (e2 > e) {
            const bool up = ((t + (uint32_t)e * T) & k) == 0;
            const unsigned long long x0 = v[e], x1 = v[e2];
            const bool sw = (x0 > x1) == up;
            v[e] = sw ? x1 : x0;
            v[e2] = sw ? x0 : x1;
          }
        }
      } else if (j < 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const unsigned long long pv = __shfl_xor_sync(FULL, v[e], j);
          const uint32_t idx = t + (uint32_t)e * T;
          const bool keep_min = ((idx & j) == 0) == ((idx & k) == 0);
          v[e] = (keep_min == (pv < v[e])) ? pv : v[e];
        }
      } else {
        unsigned long long* xb = xp ? b1 : b0;
        xp ^= 1;
#pragma unroll
        for (int e = 0; e < E; ++e) xb[t + e * T] = v[e];
        bar_named(T);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t idx = t + (uint32_t)e * T;
          const unsigned long long pv = xb[idx ^ j];
          const bool keep_min = ((idx & j) == 0) == ((idx & k) == 0);
          v[e] = (keep_min == (pv < v[e])) ? pv : v[e];
        }
      }
    }
  }
}

// Sort sbuf[0, P2) (words at mt and beyond padded with ~0) with E = P2 / NT
// words per thread; every thread of the block calls it.
template <int NT, int LOGP>
__device__ __forceinline__ void pf_sortE(unsigned long long* sbuf, unsigned long long* xch, uint32_t mt) {
  constexpr int E = (1 << LOGP) / NT;
  static_assert(E >= 2, "one word per thread has its own network");
  unsigned long long v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t idx = threadIdx.x + e * NT;
    v[e] = idx < mt ? sbuf[idx] : ~0ull;
  }
  bar_named(NT);
  bitonicE<LOGP, E>(v, sbuf, xch);
  bar_named(NT);
#pragma unroll
  for (int e = 0; e < E; ++e) sbuf[threadIdx.x + e * NT] = v[e];
}

// SORTED: sbuf already holds the instance's whole order (the full-order
// batched step); `keys` then holds the same sorted words and nkeys = their
// count (otherwise keys are slot-indexed and nkeys = MA).
template <int NT, int EM, bool SORTED = false>
__device__ void pf_finish(const Slots& S, const augsched_config& cfg, int64_t cap, uint64_t now, uint32_t inst,
                          size_t base, const unsigned long long* keys, unsigned long long* sbuf,
                          unsigned long long* xch, uint32_t mt, uint32_t target, long long B, uint32_t* order,
                          uint32_t* keyout, uint32_t* grant, uint32_t* admitted, uint32_t* gslot, SelShm& sel,
                          unsigned long long* wsum, unsigned long long& freed,
                          const unsigned long long* H = nullptr, uint32_t nH = 0, uint32_t nkeys = 0xFFFFFFFFu) {
  const int tid = threadIdx.x;
  const uint32_t MA = S.MA;
  if (nkeys == 0xFFFFFFFFu) nkeys = MA;
  // ---- bitonic sort of the prefix, padded to a power of two P2 <= EM * NT:
  // one word per thread up to P2 = NT (<= 1,024), else E = P2 / NT words per
  // thread; both networks fully unrolled per size.
  uint32_t P2 = 32;
  while (P2 < mt) P2 <<= 1;
  if (SORTED) {
  } else if (P2 <= (uint32_t)NT && P2 <= 1024u) {
    if ((uint32_t)tid < P2) {
      unsigned long long v = (uint32_t)tid < mt ? sbuf[tid] : ~0ull;
      bar_named(P2);
      switch (P2) {
        case 32: v = bitonic1<5>(v, sbuf, xch); break;
        case 64: v = bitonic1<6>(v, sbuf, xch); break;
        case 128: v = bitonic1<7>(v, sbuf, xch); break;
        case 256: v = bitonic1<8>(v, sbuf, xch); break;
        case 512: v = bitonic1<9>(v, sbuf, xch); break;
        default: v = bitonic1<10>(v, sbuf, xch); break;
      }
      bar_named(P2);
      sbuf[tid] = v;
    }
  } else if (NT == 256) {
    static_assert(NT != 256 || EM >= 4, "prefix of 1,024 words");
    if (P2 == 512) pf_sortE<256, 9>(sbuf, xch, mt);
    else pf_sortE<256, 10>(sbuf, xch, mt);
  } else if (NT == 1024) {
    static_assert(NT != 1024 || EM >= 8, "prefix of 8,192 words");
    if (P2 == 2048) pf_sortE<1024, 11>(sbuf, xch, mt);
    else if (P2 == 4096) pf_sortE<1024, 12>(sbuf, xch, mt);
    else pf_sortE<1024, 13>(sbuf, xch, mt);
  }
  __syncthreads();
  PF_T(4, false);
  const uint32_t m = target;
  // ---- a6 admission over the prefix (P_{j-1} < B, partial last, R17)
  unsigned long long Prun = 0, gsum = 0;
  uint32_t adm = 0;
  // token state of the next round's entries is loaded before this round's
  // scan (one round of lookahead hides the gather latency)
  int32_t nx_ctx = 0, nx_kv = 0, nx_cpu = 0, nx_pend = 0;
  uint32_t nx_slot = 0;
  if ((uint32_t)tid < m) {
    nx_slot = (uint32_t)sbuf[tid] & SLOT_MASK;
    const size_t g = base + nx_slot;
    nx_ctx = S.ctx[g]; nx_kv = S.kv[g]; nx_cpu = S.cpu[g]; nx_pend = S.pend[g];
  }
  for (uint32_t j0 = 0; j0 < m && (long long)Prun < B; j0 += NT) {
    const uint32_t j = j0 + tid;
    unsigned long long d = 0;
    const uint32_t slot = nx_slot;
    if (j < m) d = demand_of(nx_ctx, nx_kv, nx_cpu, nx_pend, cfg.s_in);
    if (j + NT < m) {
      nx_slot = (uint32_t)sbuf[j + NT] & SLOT_MASK;
      const size_t g = base + nx_slot;
      nx_ctx = S.ctx[g]; nx_kv = S.kv[g]; nx_cpu = S.cpu[g]; nx_pend = S.pend[g];
    }
    unsigned long long tot;
    const unsigned long long inc = block_incl_scan_u64<NT>(d, wsum, &tot);
    PF_T(7, false);
    const unsigned long long ex = Prun + inc - d;
    const bool in = j < m && (long long)ex < B;
    if (in) {
      const unsigned long long g = d < (unsigned long long)B - ex ? d : (unsigned long long)B - ex;
      order[base + j] = slot;
      keyout[base + j] = (uint32_t)(sbuf[j] >> PK_KEY);
      grant[base + j] = (uint32_t)g;
      gslot[base + slot] = (uint32_t)g;
      gsum += g;
    }
    adm += __syncthreads_count(in);
    Prun += tot;
  }
  unsigned long long need;
  block_incl_scan_u64<NT>(gsum, wsum, &need);
  PF_T(5, false);
  long long fr = cap - ld_ll(&S.A[inst]) - ld_ll(&S.P[inst]);
  // ---- a7 resolution (rare).  Candidates: every slot of the instance, or,
  // with the holder list H (single-instance prefix step), the slots that can
  // hold KV: H's running / swapped words, H's Preserve-paused slots (tier-3
  // words) and the granted waiting entries of the prefix.  Both index sets
  // give the same candidate sets, so the same selections.
  if ((long long)need > fr) {
    if (tid == 0) freed = 0;
    auto pslot = [&](uint32_t i, uint32_t& x) -> bool {
      if (!H) { x = i; return true; }
      const unsigned long long hx = H[i];
      x = (uint32_t)hx & SLOT_MASK;
      return (hx >> PK_TIER) == 3;
    };
    auto getp = [&](uint32_t i, uint64_t& key, uint32_t& w) {
      uint32_t x;
      if (!pslot(i, x)) return false;
      const uint32_t stv = S.st[base + x];
      const int32_t kv = S.kv[base + x];
      if ((stv & 15) != ST_PAUSED || ((stv >> 4) & 3) != POL_P || kv <= 0) return false;
      key = ((uint64_t)(0xFFFFFFFFu - (uint32_t)kv) << 24) | x;
      w = (uint32_t)kv;
      return true;
    };
    const uint32_t np = H ? nH : MA;
    wselect<NT>(sel, np, (uint64_t)((long long)need - fr), 56, getp);
    {
      const bool f0 = sel.r.found != 0;
      const uint64_t kd = sel.r.k;
      for (uint32_t i = tid; i < np; i += NT) {
        uint64_t key;
        uint32_t w;
        if (getp(i, key, w) && (!f0 || key <= kd)) {
          const uint32_t x = (uint32_t)key & 0xFFFFFFu;
          atomicAdd(&freed, (unsigned long long)w);
          S.kv[base + x] = 0;
          S.st[base + x] = ST_PAUSED | ((uint32_t)POL_D << 4);
        }
      }
    }
    __syncthreads();
    if (tid == 0) ledger_add(&S.P[inst], -(long long)freed);
    fr += (long long)freed;
    if ((long long)need > fr) {
      // from the tail of the order over queued entries with kv + g > 0
      auto eword = [&](uint32_t v, unsigned long long& kx) -> bool {
        if (H) {
          if (v < nH) { kx = H[v]; return (kx >> PK_TIER) < 3; }
          kx = sbuf[v - nH];           // granted entries; the running / swapped ones are in H
          return (kx >> PK_TIER) == 2;
        }
        kx = keys ? keys[v]
                  : slot_word(S.coef[inst], S.ip[inst], S.st[base + v], S.V[base + v], S.last[base + v], now, v);
        return (kx >> PK_TIER) < 3;
      };
      auto gete = [&](uint32_t v, uint64_t& key, uint32_t& w) {
        unsigned long long kx;
        if (!eword(v, kx)) return false;
        const uint32_t x = (uint32_t)kx & SLOT_MASK;
        const uint32_t g = gslot[base + x];
        w = (uint32_t)S.kv[base + x] + (g == 0xFFFFFFFFu ? 0u : g);
        key = ~kx;
        return w > 0;
      };
      const uint32_t ne = H ? nH + adm : nkeys;
      wselect<NT>(sel, ne, (uint64_t)((long long)need - fr), 64, gete);
      const bool f1 = sel.r.found != 0;
      const uint64_t k1 = sel.r.k;
      __syncthreads();
      long long dA = 0;
      for (uint32_t v = tid; v < ne; v += NT) {
        uint64_t key;
        uint32_t w;
        if (gete(v, key, w) && (!f1 || key <= k1)) {
          const uint32_t x = (uint32_t)~key & SLOT_MASK;
          dA -= S.kv[base + x];
          S.kv[base + x] = 0;
          S.cpu[base + x] = 0;
          S.st[base + x] = ST_WAIT | (S.st[base + x] & 0x30u);
          mark_dirty(S, (uint32_t)(base + x), S.ti_ep + 1);   // its word changes (tier)
          if (gslot[base + x]) gslot[base + x] = 0xFFFFFFFFu;   // grant cancelled
        }
      }
      if (dA) ledger_add(&S.A[inst], dA);
      __syncthreads();
      for (uint32_t j = tid; j < adm; j += NT)
        if (gslot[base + order[base + j]] == 0xFFFFFFFFu) grant[base + j] = 0;
    }
  }
  __syncthreads();
  PF_T(6, false);
  // ---- S9 + token accounting of the granted batch
  unsigned long long dA = 0;
  for (uint32_t j = tid; j < adm; j += NT) {
    const size_t g_slot = base + order[base + j];
    gslot[g_slot] = 0;
    const uint32_t gr = grant[base + j];
    if (gr == 0) continue;
    int32_t ctx = S.ctx[g_slot], kv = S.kv[g_slot], cpu = S.cpu[g_slot], pend = S.pend[g_slot];
    if (cpu > 0) { cpu -= (int32_t)gr; kv += (int32_t)gr; }
    else if ((ctx - kv) + pend > 0) {
      const int32_t rc = (int32_t)gr < ctx - kv ? (int32_t)gr : ctx - kv;
      kv += rc;
      const int32_t pp = (int32_t)gr - rc;
      pend -= pp; ctx += pp; kv += pp;
    } else { ctx += 1; kv += 1; }
    dA += gr;
    S.ctx[g_slot] = ctx; S.kv[g_slot] = kv; S.cpu[g_slot] = cpu; S.pend[g_slot] = pend;
    S.last[g_slot] = (uint32_t)now;
    S.st[g_slot] = ST_RUN | (S.st[g_slot] & 0x30u);
    mark_dirty(S, (uint32_t)g_slot, S.ti_ep + 1);   // last and tier change
  }
  unsigned long long tot;
  block_incl_scan_u64<NT>(dA, wsum, &tot);
  if (tid == 0) {
    admitted[inst] = adm;
    if (S.gdirty[inst] < adm) S.gdirty[inst] = adm;
    const long long a = ld_ll(&S.A[inst]) + (long long)tot;
    S.A[inst] = a;
    S.Aevt[inst] = a;
#ifdef AUGSCHED_DEBUG
    debug_check_step(S, inst, tot, B, cap);
#endif
  }
}

// ---- single-instance prefix step (see the comment above pf_target)
enum : int {
  PC_A = 0, PC_C, PC_BSTAR, PC_BELOW, PC_SPEC, PC_ARR1, PC_STATE, PC_ARR2, PC_REL2, PC_ARR3, PC_TARGET, PC_H,
  PF_NCNT = 16
};
constexpr uint32_t PF_HCAP = 65536;   // holder-list capacity (running, swapped, Preserve-paused slots)
constexpr int FNT = 1024;   // threads per CTA
#ifndef AUGSCHED_PF_KU
#define AUGSCHED_PF_KU 8
#endif
constexpr int FKU = AUGSCHED_PF_KU;   // slots in flight per thread

struct PfArgs {
  Slots S;
  augsched_config cfg;
  int64_t cap;
  uint64_t now;
  uint32_t N;
  int spec;                       // 1: phase 1 (speculative pass) first
  unsigned long long* k0;         // [N] packed words (fallback)
  unsigned long long* A;          // [PF_SCAP] phase-1 candidates, then words below b*
  unsigned long long* C;          // [N] words in b*
  unsigned long long* theta;      // [2] anchor word, anchor slot (kept across steps)
  unsigned long long* H;          // [PF_HCAP] words of the slots that can hold KV (resolution candidates)
  uint32_t* ghist;                // [1 << PF_BITS]
  uint32_t* cnt;                  // [PF_NCNT]: append counts (zero at entry, zeroed again by the
                                  // finishing CTA), arrival counts (cumulative, mod G), epoch-tagged flags
  uint32_t ep;                    // this call's epoch tag (1 .. 2^30 - 1)
  uint32_t* n_active;             // this call's queue-size word (zero at entry)
  uint32_t* n_active_next;        // the other one: the previous call's output, zeroed for the next call
  long long* budget;
  uint32_t *order, *keyout, *grant, *admitted, *gslot;
};

__device__ __forceinline__ uint32_t vld(const uint32_t* p) { return *(volatile const uint32_t*)p; }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// candidates kept beyond the prefix for the next step's anchor
__device__ __forceinline__ uint32_t pf_margin(uint32_t target) { return target / 2 > 256u ? target / 2 : 256u; }

// Arrive at a grid-wide counter; true in the CTA that arrives last.  The
// caller's global writes are visible to that CTA.
// Arrive at a grid-wide counter; true in the CTA that arrives last.  The
// counter is never reset: every call adds exactly G arrivals, so the last
// arrival is the one that makes it a multiple of G.
__device__ __forceinline__ bool pf_arrive_last(uint32_t* ctr, uint32_t G, uint32_t& flag) {
  __syncthreads();   // the CTA's writes happen before thread 0's release (cumulative fence)
  if (threadIdx.x == 0) {
    __threadfence();
    flag = (atomicAdd(ctr, 1u) + 1u) % G == 0;
    if (flag) __threadfence();
  }
  __syncthreads();
  const bool last = flag != 0;
  __syncthreads();   // every thread has read `flag` before thread 0 may reuse it
  return last;
}

// Epoch-tagged flag word: (epoch << 2) | value.  Wait until this call's
// epoch shows; returns the value.
__device__ __forceinline__ void pf_post(uint32_t* w, uint32_t ep, uint32_t v) {
  __threadfence();
  atomicExch(w, (ep << 2) | v);
}
__device__ __forceinline__ uint32_t pf_wait(const uint32_t* w, uint32_t ep, uint32_t& flag) {
  if (threadIdx.x == 0) {
    uint32_t v;
    while (((v = vld(w)) >> 2) != ep) __nanosleep(32);
    flag = v & 3u;
  }
  __syncthreads();
  const uint32_t r = flag;
  __syncthreads();   // every thread has read `flag` before thread 0 may reuse it
  return r;
}


__global__ void __launch_bounds__(FNT, 1) pf_step_kernel(const __grid_constant__ PfArgs a) {
  extern __shared__ __align__(16) unsigned long long pf_sm[];
  unsigned long long* sbuf = pf_sm;   // [2 * PF_SCAP]: the prefix + the sort's exchange buffer
  constexpr int NB = 1 << PF_BITS;
  __shared__ uint32_t h[NB];
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[FNT / 32 + 1];
  __shared__ unsigned long long freed, th_s;
  __shared__ uint32_t m_s, flag_s, q_s;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t G = gridDim.x, N = a.N;
  const Slots& S = a.S;
  const Coef k = S.coef[0];
  const augsched_instance_params ip = S.ip[0];
  const unsigned lt = (1u << lane) - 1;
  // a contiguous range of slots per CTA (one pass of FKU loads per thread at 1 M slots)
  const uint32_t chunk = ((N + G - 1) / G + 31) & ~31u;
  const uint32_t c0 = blockIdx.x * chunk < N ? blockIdx.x * chunk : N;
  const uint32_t c1 = c0 + chunk < N ? c0 + chunk : N;
  uint32_t* cnt = a.cnt;
  PF_T(0, true);
  PF_T(1, false);
  __shared__ long long B_s;
  __shared__ uint32_t tgt_s, nH_s, wkv_s;
  auto finish = [&](uint32_t mt, const unsigned long long* keys) {
    const long long B = B_s;
    const uint32_t target = tgt_s, nH = nH_s;
    PF_T(3, false);
    const bool use_h = nH <= PF_HCAP && wkv_s == 0;
    pf_finish<FNT, PF_SCAP / FNT>(S, a.cfg, a.cap, a.now, 0, 0, keys, sbuf, sbuf + PF_SCAP, mt, target, B,
                                  a.order, a.keyout, a.grant, a.admitted, a.gslot, sel, wsum, freed,
                                  use_h ? a.H : nullptr, nH);
    // next anchor: the K-th smallest word, K a margin beyond the prefix
    if (tid == 0) {
      const uint32_t K = target + pf_margin(target) < mt ? target + pf_margin(target) : mt;
#ifdef AUGSCHED_PF_TIMING
      const unsigned long long t5 = gtime();
      printf("pf_t state %u mt %u target %u nH %u K %u | ns: start..%llu arrive %llu finish %llu sorted %llu "
             "admitted %llu resolved %llu end %llu\n", __ldcg(&cnt[PC_STATE]), mt, target, __ldcg(&cnt[PC_H]), K,
             g_pf_t[1] - g_pf_t[0], g_pf_t[2] - g_pf_t[0], g_pf_t[3] - g_pf_t[0], g_pf_t[4] - g_pf_t[0],
             g_pf_t[5] - g_pf_t[0], g_pf_t[6] - g_pf_t[0], t5 - g_pf_t[0]);
      printf("pf_t gathered+scanned %llu\n", g_pf_t[7] - g_pf_t[0]);
      g_pf_t[0] = ~0ull;
      for (int q = 1; q < 8; ++q) g_pf_t[q] = 0;
#endif
      a.theta[0] = K > 0 ? sbuf[K - 1] : ~0ull;
      a.theta[1] = K > 0 ? (sbuf[K - 1] & SLOT_MASK) : ~0ull;
      // every other CTA is done with the append counters: clear them (and the
      // next call's queue-size word) for the next call
      cnt[PC_SPEC] = 0; cnt[PC_H] = 0; cnt[PC_A] = 0; cnt[PC_C] = 0;
      *a.n_active_next = 0;
    }
  };
  // slots that can hold KV: running, swapped, Preserve-paused (the
  // resolution candidates besides the granted waiting entries)
  auto add_holder = [&](uint32_t stv, unsigned long long w, bool valid) {
    const uint32_t s4 = stv & 15;
    const bool hold = valid && (s4 == ST_RUN || s4 == ST_SWAP || (s4 == ST_PAUSED && ((stv >> 4) & 3) == POL_P));
    const unsigned m = __ballot_sync(FULL, hold);
    if (m) {
      const int ld = __ffs(m) - 1;
      uint32_t b = 0;
      if (lane == ld) b = atomicAdd(&cnt[PC_H], (unsigned)__popc(m));
      b = __shfl_sync(FULL, b, ld) + __popc(m & lt);
      if (hold && b < PF_HCAP) a.H[b] = w;
    }
  };
  auto count_queued = [&](uint32_t myq) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) myq += __shfl_xor_sync(FULL, myq, o);
    if (tid == 0) q_s = 0;
    __syncthreads();
    if (lane == 0 && myq) atomicAdd(&q_s, myq);
    __syncthreads();
    if (tid == 0 && q_s) atomicAdd(a.n_active, q_s);
  };
  // target = min(B, n) once the queue size is complete (last CTA only)
  // thread 0 of the deciding CTA: limit, target = min(B, n), holder count
  // (independent loads issued together)
  auto set_target = [&]() -> uint32_t {
    const long long A0 = __ldcg(&S.A[0]), P0 = __ldcg(&S.P[0]);
    const uint32_t nq = __ldcg(a.n_active), nh = __ldcg(&cnt[PC_H]), wk = __ldcg(S.wkv);
    const long long B = token_limit(a.cfg, k, ip, a.cap, A0, P0);
    const uint32_t target = pf_target(B, nq);
    a.budget[0] = B;
    cnt[PC_TARGET] = target;
    B_s = B; tgt_s = target; nH_s = nh; wkv_s = wk;
    return target;
  };

  if (a.spec) {
    // ---- phase 1: speculative pass against the anchor word
    unsigned long long th = 0;
    bool have_th = false;
    uint32_t myq = 0;
    for (uint32_t b0 = c0; b0 < c1; b0 += FNT * FKU) {   // block-uniform trip count
      uint32_t stv[FKU], lst[FKU];
      double V[FKU];
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t s = b0 + u * FNT + tid;
        stv[u] = 0u; lst[u] = 0u; V[u] = 0.0;
        if (s < c1) { stv[u] = S.st[s]; V[u] = S.V[s]; lst[u] = S.last[s]; }
      }
      if (!have_th) {
        // the anchor's current word, fetched while the first loads are in flight
        if (tid == 0) {
          unsigned long long t0 = a.theta[0];
          const unsigned long long sg = a.theta[1];
          if (sg < N) {
            const unsigned long long w = slot_word(k, ip, S.st[sg], S.V[sg], S.last[sg], a.now, (uint32_t)sg);
            if ((w >> PK_TIER) < 3) t0 = w;
          }
          th_s = t0;
        }
        __syncthreads();
        th = th_s;
        have_th = true;
      }
      // words, then one atomic per warp and list for all its appends (the
      // holders and candidates cluster in a few CTAs: per-item atomics would
      // chain their round trips)
      unsigned long long wv[FKU];
      unsigned cm[FKU], hm[FKU];
      uint32_t nc = 0, nh = 0;
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t s = b0 + u * FNT + tid;
        const unsigned long long w = slot_word(k, ip, stv[u], V[u], lst[u], a.now, s);
        const bool q = s < c1 && (w >> PK_TIER) < 3;
        const uint32_t s4 = stv[u] & 15;
        const bool hold = s < c1 && (s4 == ST_RUN || s4 == ST_SWAP ||
                                     (s4 == ST_PAUSED && ((stv[u] >> 4) & 3) == POL_P));
        myq += q;
        wv[u] = w;
        cm[u] = __ballot_sync(FULL, q && w <= th);
        hm[u] = __ballot_sync(FULL, hold);
        nc += __popc(cm[u]);
        nh += __popc(hm[u]);
      }
      if (nc | nh) {
        uint32_t bc = 0, bh = 0;
        if (lane == 0) {
          if (nc) bc = atomicAdd(&cnt[PC_SPEC], nc);
          if (nh) bh = atomicAdd(&cnt[PC_H], nh);
        }
        bc = __shfl_sync(FULL, bc, 0);
        bh = __shfl_sync(FULL, bh, 0);
#pragma unroll
        for (int u = 0; u < FKU; ++u) {
          const uint32_t s = b0 + u * FNT + tid;
          if ((cm[u] >> lane) & 1u) {
            const uint32_t b = bc + __popc(cm[u] & lt);
            if (b < PF_SCAP) {
              a.A[b] = wv[u];
#ifndef AUGSCHED_PF_NO_PREFETCH
              // the admission reads this slot's token state: start bringing it to L2
              prefetch_l2(&S.ctx[s]); prefetch_l2(&S.kv[s]); prefetch_l2(&S.cpu[s]); prefetch_l2(&S.pend[s]);
#endif
            }
          }
          if ((hm[u] >> lane) & 1u) {
            const uint32_t b = bh + __popc(hm[u] & lt);
            if (b < PF_HCAP) a.H[b] = wv[u];
          }
          bc += __popc(cm[u]);
          bh += __popc(hm[u]);
        }
      }
    }
    count_queued(myq);
    PF_T(2, false);
    if (pf_arrive_last(&cnt[PC_ARR1], G, flag_s)) {
      if (tid == 0) {
        const uint32_t nc = __ldcg(&cnt[PC_SPEC]);
        const uint32_t target = set_target();
        const bool ok = target == 0 || (nc >= target && nc <= PF_SCAP);
        m_s = ok ? (target == 0 ? 0u : nc) : 0xFFFFFFFFu;
        pf_post(&cnt[PC_STATE], a.ep, ok ? 1u : 2u);
      }
      __syncthreads();
      const uint32_t mt = m_s;
      if (mt != 0xFFFFFFFFu) {
        for (uint32_t i = tid; i < mt; i += FNT) sbuf[i] = __ldcg(&a.A[i]);
        __syncthreads();
        finish(mt, nullptr);
        return;
      }
    } else if (pf_wait(&cnt[PC_STATE], a.ep, flag_s) == 1) {
      return;
    }
  }
  // ---- phase 2: packed words + histogram of the top digit
  for (int b = tid; b < NB; b += FNT) h[b] = 0;
  __syncthreads();
  {
    uint32_t myq = 0;
    for (uint32_t b0 = c0; b0 < c1; b0 += FNT * FKU) {
      uint32_t stv[FKU], lst[FKU];
      double V[FKU];
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t s = b0 + u * FNT + tid;
        stv[u] = 0u; lst[u] = 0u; V[u] = 0.0;
        if (s < c1) { stv[u] = S.st[s]; V[u] = S.V[s]; lst[u] = S.last[s]; }
      }
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t s = b0 + u * FNT + tid;
        const unsigned long long w = slot_word(k, ip, stv[u], V[u], lst[u], a.now, s);
        const bool q = s < c1 && (w >> PK_TIER) < 3;
        if (s < c1) a.k0[s] = w;
        if (!a.spec) add_holder(stv[u], w, s < c1);
        myq += q;
        hist_add(h, q ? (int)(w >> (64 - PF_BITS)) : -1);
      }
    }
    __syncthreads();
    for (int b = tid; b < NB; b += FNT)
      if (h[b]) atomicAdd(&a.ghist[b], h[b]);
    if (!a.spec) count_queued(myq);
  }
  if (pf_arrive_last(&cnt[PC_ARR2], G, flag_s)) {
    // locate b*: the bucket holding the target-th word
    __shared__ uint32_t tgt2_s, wtot[FNT / 32];
    if (tid == 0) tgt2_s = a.spec ? __ldcg(&cnt[PC_TARGET]) : set_target();
    __syncthreads();
    const uint32_t target = tgt2_s;
    constexpr int PER = NB / FNT;
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      loc[j] = __ldcg(&a.ghist[tid * PER + j]);
      sum += loc[j];
      a.ghist[tid * PER + j] = 0;   // all CTAs have added theirs: clear for the next call
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[tid >> 5] = inc;
    if (tid == 0) { cnt[PC_BSTAR] = NB; cnt[PC_BELOW] = 0; }
    __syncthreads();
    uint32_t run = inc - sum;
    for (int w = 0; w < (tid >> 5); ++w) run += wtot[w];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (target > 0 && run < target && run + loc[j] >= target) { cnt[PC_BSTAR] = tid * PER + j; cnt[PC_BELOW] = run; }
      run += loc[j];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) pf_post(&cnt[PC_REL2], a.ep, 1u);
  } else {
    pf_wait(&cnt[PC_REL2], a.ep, flag_s);
  }
  // ---- phase 3: words below b* -> A, in b* -> C
  const uint32_t bstar = __ldcg(&cnt[PC_BSTAR]);
  if (bstar < NB) {
    for (uint32_t b0 = c0; b0 < c1; b0 += FNT * FKU) {
      unsigned long long x[FKU];
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t s = b0 + u * FNT + tid;
        x[u] = s < c1 ? __ldcg(&a.k0[s]) : ~0ull;
      }
#pragma unroll
      for (int u = 0; u < FKU; ++u) {
        const uint32_t d = (uint32_t)(x[u] >> (64 - PF_BITS));
        const bool queued = (x[u] >> PK_TIER) < 3;
        const bool inA = queued && d < bstar, inC = queued && d == bstar;
        const unsigned ma = __ballot_sync(FULL, inA), mc = __ballot_sync(FULL, inC);
        if (!(ma | mc)) continue;
        uint32_t ba = 0, bc = 0;
        if (lane == 0) {
          if (ma) ba = atomicAdd(&cnt[PC_A], (unsigned)__popc(ma));
          if (mc) bc = atomicAdd(&cnt[PC_C], (unsigned)__popc(mc));
        }
        ba = __shfl_sync(FULL, ba, 0);
        bc = __shfl_sync(FULL, bc, 0);
        if (inA) a.A[ba + __popc(ma & lt)] = x[u];
        if (inC) a.C[bc + __popc(mc & lt)] = x[u];
      }
    }
  }
  if (!pf_arrive_last(&cnt[PC_ARR3], G, flag_s)) return;
  // ---- the last CTA: the first `target` words (+ a margin) and the finish
  if (tid == 0) {
    const uint32_t nq = __ldcg(a.n_active), nh = __ldcg(&cnt[PC_H]), wk = __ldcg(S.wkv);
    const long long B = ld_ll(a.budget);
    B_s = B; tgt_s = pf_target(B, nq); nH_s = nh; wkv_s = wk;
  }
  __syncthreads();
  const uint32_t target = tgt_s;
  const uint32_t nA = __ldcg(&cnt[PC_A]), nC = __ldcg(&cnt[PC_C]);
  for (uint32_t i = tid; i < nA; i += FNT) sbuf[i] = __ldcg(&a.A[i]);
  if (tid == 0) m_s = nA;
  uint32_t needC = target > nA ? target - nA : 0u;
  if (needC > 0 && nA + nC <= PF_SCAP) {
    // the whole crossing bucket fits beside A
    for (uint32_t i = tid; i < nC; i += FNT) sbuf[nA + i] = __ldcg(&a.C[i]);
    if (tid == 0) m_s = nA + nC;
  } else if (needC > 0) {
    // large crossing bucket: its needC (+ margin) smallest
    needC += pf_margin(target);
    needC = needC < nC ? needC : nC;
    needC = needC < PF_SCAP - nA ? needC : PF_SCAP - nA;
    const unsigned long long* cb = a.C;
    __syncthreads();
    wselect<FNT>(sel, nC, needC, 64, [&](uint32_t i, uint64_t& key, uint32_t& w) {
      key = __ldcg(&cb[i]); w = 1u; return true; });
    const unsigned long long tau = sel.r.found ? sel.r.k : ~0ull;
    for (uint32_t i = tid; i < nC; i += FNT) {
      const unsigned long long x = __ldcg(&cb[i]);
      if (x <= tau) sbuf[atomicAdd(&m_s, 1u)] = x;
    }
  }
  __syncthreads();
  finish(m_s, a.k0);
}


// Prefix step of a multi-instance handle: one CTA per instance keeps the
// instance's packed words in shared memory, selects its first min(B, n)
// order entries by a count-weighted radix select, then pf_finish.
template <int NT, int EM>
__global__ void __launch_bounds__(NT) pf_multi_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                       long long* budget, uint32_t* n_active, uint32_t* order,
                                                       uint32_t* keyout, uint32_t* grant, uint32_t* admitted,
                                                       uint32_t* gslot, uint32_t sbuf_cap,
                                                       unsigned long long* theta) {
  extern __shared__ __align__(16) unsigned long long pf_sm[];
  const uint32_t MA = S.MA;
  unsigned long long* kbuf = pf_sm;             // [MA] packed words of the instance
  unsigned long long* sbuf = pf_sm + MA;        // [sbuf_cap] the prefix
  unsigned long long* xch = sbuf + sbuf_cap;    // [sbuf_cap] sort exchange buffer
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[NT / 32 + 1];
  __shared__ unsigned long long freed;
  __shared__ uint32_t m_s, c_s;
  __shared__ long long B_s;
  __shared__ unsigned long long th_s;
  const int tid = threadIdx.x;
  const uint32_t inst = blockIdx.x;
  const size_t base = (size_t)inst * MA;
  const Coef& k = S.coef[inst];
  const augsched_instance_params& ip = S.ip[inst];
  if (tid == 0) {
    B_s = token_limit(cfg, k, ip, cap, ld_ll(&S.A[inst]), ld_ll(&S.P[inst]));
    budget[inst] = B_s;
    m_s = 0;
    c_s = 0;
  }
  unsigned long long myq = 0;
  {
    // 8 slots per thread loaded together, every field unconditionally (one
    // round trip per 8 slots instead of two dependent ones per slot)
    constexpr int UE = 8;
    const Coef kr = k;
    for (uint32_t x0 = 0; x0 < MA; x0 += (uint32_t)NT * UE) {
      uint32_t stv[UE], lst[UE];
      double V[UE];
#pragma unroll
      for (int e = 0; e < UE; ++e) {
        const uint32_t x = x0 + (uint32_t)e * NT + tid;
        stv[e] = 0u; lst[e] = 0u; V[e] = 0.0;
        if (x < MA) { stv[e] = S.st[base + x]; V[e] = S.V[base + x]; lst[e] = S.last[base + x]; }
      }
#pragma unroll
      for (int e = 0; e < UE; ++e) {
        const uint32_t x = x0 + (uint32_t)e * NT + tid;
        if (x < MA) {
          const unsigned long long w = slot_word(kr, ip, stv[e], V[e], lst[e], now, x);
          kbuf[x] = w;
          myq += (w >> PK_TIER) < 3;
        }
      }
    }
  }
  unsigned long long nq;
  block_incl_scan_u64<NT>(myq, wsum, &nq);   // syncs
  const long long B = B_s;
  const uint32_t target = pf_target(B, (uint32_t)nq);
  if (tid == 0) n_active[inst] = (uint32_t)nq;
  // candidates kept beyond the prefix (the anchor's margin), within the buffer
  const uint32_t margin = target / 8 > 32u ? target / 8 : 32u;
  uint32_t want = target + margin < (uint32_t)nq ? target + margin : (uint32_t)nq;
  want = want < sbuf_cap ? want : sbuf_cap;
  if (target > 0) {
    // anchored filter (as in the single-instance step): the words at or below
    // the current word of the slot the previous step chose a margin beyond its
    // prefix; exact whenever target <= their count <= sbuf_cap.  Otherwise
    // (first step, random ranking, events that moved the anchor) a
    // count-weighted radix select of the `want` smallest.
    if (tid == 0) {
      unsigned long long th = 0;   // no anchor: take the select
      if (ip.ranking != AUGSCHED_RANK_RANDOM) {
        th = theta[2 * inst];
        const unsigned long long sg = theta[2 * inst + 1];
        if (sg < MA && (kbuf[sg] >> PK_TIER) < 3) th = kbuf[sg];
      }
      th_s = th;
    }
    __syncthreads();
    const unsigned long long th = th_s;
    uint32_t c = 0;
    for (uint32_t x = tid; x < MA; x += NT) {
      const unsigned long long kx = kbuf[x];
      c += (kx >> PK_TIER) < 3 && kx <= th;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((tid & 31) == 0 && c) atomicAdd(&c_s, c);
    __syncthreads();
    const uint32_t cnt = c_s;
    unsigned long long tau = th;
    if (cnt < target || cnt > sbuf_cap) {
      wselect<NT>(sel, MA, want, 64, [&](uint32_t i, uint64_t& key, uint32_t& w) {
        key = kbuf[i]; w = 1u; return (key >> PK_TIER) < 3; });
      tau = sel.r.found ? sel.r.k : ~0ull;
    }
    for (uint32_t x = tid; x < MA; x += NT) {
      const unsigned long long kx = kbuf[x];
      if ((kx >> PK_TIER) < 3 && kx <= tau) sbuf[atomicAdd(&m_s, 1u)] = kx;
    }
  }
  __syncthreads();
  const uint32_t mt = m_s;
  pf_finish<NT, EM>(S, cfg, cap, now, inst, base, kbuf, sbuf, xch, mt, target, B, order, keyout, grant,
                    admitted, gslot, sel, wsum, freed);
  // next anchor: the want-th smallest word (sbuf is sorted by pf_finish)
  if (tid == 0) {
    const uint32_t K = want < mt ? want : mt;
    theta[2 * inst] = K > 0 ? sbuf[K - 1] : ~0ull;
    theta[2 * inst + 1] = K > 0 ? (sbuf[K - 1] & SLOT_MASK) : ~0ull;
  }
}


// Full-order step of a multi-instance handle (the batched scheduler): one CTA
// per instance sorts all of the instance's packed words in shared memory --
// a stable LSD radix sort of the 34-bit (tier, key) field above the slot
// (digits of 9, 9, 8 and 8 bits), each warp ranking a contiguous run of
// E x 32 words with ballot-built digit-peer masks and warp-private digit
// counters, one block scan of the (digit, warp) counters per pass -- then
// admission / resolution / grant accounting (pf_finish over the sorted
// words), and writes the whole order, keys, zero grants beyond the prefix,
// the queue size and the per-tier segment starts.  Words of slots that are
// not queued carry tier 3 and sort behind the queue.  No device-wide pass:
// HBM traffic is the 16 B/slot read of the scoring state plus the 12 B/slot
// order/key/grant write.

#ifndef AUGSCHED_FM_MATCH
#define AUGSCHED_FM_MATCH 0   // 1: __match_any_sync digit peers instead of bit ballots
#endif
#ifndef AUGSCHED_FM_MINB
#define AUGSCHED_FM_MINB 4     // resident CTAs per SM the register budget targets (256 threads, E = 8; 5 spills: slower)
#endif
constexpr uint32_t FM_DCAP = 1024;   // incremental order: out-of-place / changed words merged (else a full sort)
#ifdef AUGSCHED_FM_TIMING
// per-phase clocks of full_multi_kernel summed over CTAs: [0..5] phases,
// [8] CTAs, [9] CTAs that merged incrementally, [10] sum of |D| there
__device__ unsigned long long g_fm_t[16];
#define FMT(i) do { if (threadIdx.x == 0) { const long long c_ = clock64(); atomicAdd(&g_fm_t[i], (unsigned long long)(c_ - fm_c)); fm_c = c_; } } while (0)
#else
#define FMT(i) do {} while (0)
#endif

// Block-wide exclusive scans over NT threads (every thread calls; two
// __syncthreads).  Max of u64 (identity 0) and sum of u32.
template <int NT>
__device__ __forceinline__ unsigned long long block_excl_max(unsigned long long v, unsigned long long* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o && y > inc) inc = y;
  }
  if (lane == 31) tmp[warp] = inc;
  __syncthreads();
  unsigned long long run = 0;
  for (int w = 0; w < warp; ++w) run = tmp[w] > run ? tmp[w] : run;
  unsigned long long ex = __shfl_up_sync(FULL, inc, 1);
  if (lane == 0) ex = 0;
  __syncthreads();
  return ex > run ? ex : run;
}
template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* tmp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) tmp[warp] = inc;
  __syncthreads();
  uint32_t run = 0, tot = 0;
  for (int w = 0; w < NT / 32; ++w) { if (w < warp) run += tmp[w]; tot += tmp[w]; }
  total = tot;
  __syncthreads();
  return run + inc - v;
}
// Entries of the sorted a[0, n) below x.
__device__ __forceinline__ uint32_t lower_rank(const unsigned long long* a, uint32_t n, unsigned long long x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int NT, int E>
__global__ void __launch_bounds__(NT, (NT == 256 && E == 8) ? AUGSCHED_FM_MINB : 1) full_multi_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                        long long* budget, uint32_t* n_active, uint32_t* tier_off,
                                                        uint32_t* order, uint32_t* keyout, uint32_t* grant,
                                                        uint32_t* admitted, uint32_t* gslot,
                                                        uint32_t* mord, uint32_t* mord_n, int inc) {
  constexpr int NW = NT / 32;
  constexpr int NBMAX = 512;
  constexpr uint32_t MP = (uint32_t)NT * E;      // padded slot count (>= MA)
  extern __shared__ __align__(16) unsigned long long fm_sm[];
  unsigned long long* buf0 = fm_sm;               // [MP]
  unsigned long long* buf1 = fm_sm + MP;          // [MP]
  // 16-bit digit counters, warp-major [NW][NBMAX] (counts and offsets < 2^16)
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(fm_sm + 2 * (size_t)MP);
  // the rare resolution's selection state reuses the counters' space (the
  // region is sized for the larger of the two, full_multi_smem)
  SelShm& sel = *reinterpret_cast<SelShm*>(wcnt);
  __shared__ unsigned long long wsum[NW + 1];
  __shared__ unsigned long long freed;
  __shared__ uint32_t tc_s[3], tsum[NT / 32];
  __shared__ long long B_s;
  __shared__ uint32_t chgb[MP / 32];              // incremental order: slot changed since the last step
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1;
  const uint32_t inst = blockIdx.x;
  const uint32_t MA = S.MA;
  const size_t base = (size_t)inst * MA;
  const Coef k = S.coef[inst];
  const augsched_instance_params ip = S.ip[inst];
  // uniform: the incremental order is tried when the previous step left this
  // handle's order (the host's flag) and the ranking is not a fresh shuffle
  const bool inc_try = inc && S.dmark && ip.ranking != AUGSCHED_RANK_RANDOM;
#ifdef AUGSCHED_FM_TIMING
  long long fm_c = clock64();
  if (tid == 0) atomicAdd(&g_fm_t[8], 1ull);
#endif
  if (tid == 0) tc_s[0] = tc_s[1] = tc_s[2] = 0;
  __syncthreads();   // the tier counters are clear before any warp adds to them
  // ---- words of every slot (a4), per-tier counts
  uint32_t tcount[3] = {0u, 0u, 0u};
  {
    // the E slots of this thread loaded together (independent loads in flight),
    // with their dirty marks when the incremental order is tried
    uint32_t stv[E], lst[E], dm[E];
    double V[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t x = tid + e * NT;
      stv[e] = 0u; lst[e] = 0u; V[e] = 0.0; dm[e] = 0u;
      if (x < MA) {
        stv[e] = S.st[base + x]; V[e] = S.V[base + x]; lst[e] = S.last[base + x];
        if (inc && S.dmark) dm[e] = __ldcg(&S.dmark[base + x]);   // kernel arguments only: no wait for ip
      }
    }
    if (tid == 0) {   // the limit's ledger loads overlap the slot loads
      B_s = token_limit(cfg, k, ip, cap, ld_ll(&S.A[inst]), ld_ll(&S.P[inst]));
      budget[inst] = B_s;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t x = tid + e * NT;
      unsigned long long w = ~0ull;
      if (x < MA) {
        w = slot_word(k, ip, stv[e], V[e], lst[e], now, x);
        const uint32_t t = (uint32_t)(w >> PK_TIER);
        if (t < 3) ++tcount[t];
      }
      buf0[x] = w;
    }
    if (inc_try) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t x = tid + e * NT;
        const bool c = x < MA && dm[e] == S.ti_ep;
        const unsigned b = __ballot_sync(FULL, c);
        if (lane == 0) chgb[(warp * 32 + e * NT) / 32] = b;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    uint32_t c = tcount[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if (lane == 0 && c) atomicAdd(&tc_s[t], c);
  }
  // ---- incremental order (rankings with an order that persists: the value
  // order of Eq.26 under R3 or B12, FCFS).  The previous step's order of this
  // instance minus the slots changed since then (dirty marks: records,
  // grants, evictions) and minus the unchanged words that are now out of
  // place (not above the running maximum of the unchanged words before them:
  // under R3 every waiting score moves by the same alpha*T per step, so only
  // rounding to fp32 reorders them) is sorted (K); the rest (D) is sorted
  // here and merged in by rank.  The result is the sorted order of the same
  // words, so it equals the full sort's; the full sort runs instead when D
  // does not fit its buffer (or the counts disagree).
  __syncthreads();   // tier counters and the changed bitmap are complete
  FMT(0);
  bool inc_ok = false;
  if (inc_try) {
    unsigned long long* dbuf = reinterpret_cast<unsigned long long*>(wcnt);   // [FM_DCAP]
    const uint32_t m = mord_n[inst];
    const uint32_t nq = tc_s[0] + tc_s[1] + tc_s[2];
    auto chg = [&](uint32_t x) { return (chgb[x >> 5] >> (x & 31)) & 1u; };
    // this thread's E consecutive positions of the previous order: the
    // unchanged queued words (0 marks a changed or departed slot)
    unsigned long long pw[E];
    unsigned long long tmax = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t j = (uint32_t)tid * E + e;
      uint32_t x = j < MA ? __ldcg(&mord[base + j]) : INVALID_SLOT;   // not waiting for m
      if (j >= m) x = INVALID_SLOT;
      pw[e] = 0;
      if (x < MA && !chg(x)) {
        const unsigned long long w = buf0[x];
        if ((uint32_t)(w >> PK_TIER) < 3) pw[e] = w;
      }
      tmax = pw[e] > tmax ? pw[e] : tmax;
    }
    unsigned long long run = block_excl_max<NT>(tmax, wsum);
    uint32_t keepm = 0, outm = 0, chm = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (pw[e]) {
        if (pw[e] > run) { keepm |= 1u << e; run = pw[e]; }
        else outm |= 1u << e;
      }
      const uint32_t x = tid + e * NT;
      if (x < MA && chg(x) && (uint32_t)(buf0[x] >> PK_TIER) < 3) chm |= 1u << e;
    }
    uint32_t KD = 0;   // both counts in one scan: kept << 16 | D (each <= 8,192)
    const uint32_t ofs = block_excl_sum<NT>(((uint32_t)__popc(keepm) << 16) | (uint32_t)(__popc(outm) + __popc(chm)),
                                            tsum, KD);
    const uint32_t kofs0 = ofs >> 16, dofs0 = ofs & 0xFFFFu, Kt = KD >> 16, Dt = KD & 0xFFFFu;
    if (Dt <= FM_DCAP && Kt + Dt == nq) {   // uniform
      uint32_t ko = kofs0, d0 = dofs0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if ((keepm >> e) & 1u) buf1[ko++] = pw[e];
        if ((outm >> e) & 1u) dbuf[d0++] = pw[e];
        if ((chm >> e) & 1u) dbuf[d0++] = buf0[tid + e * NT];
      }
      __syncthreads();   // buf0 is no longer read: it serves the sort's exchange, then holds the order
      uint32_t P2 = 32;
      while (P2 < Dt) P2 <<= 1;
      if (Dt > 1) {
        if (P2 <= (uint32_t)NT) {
          if ((uint32_t)tid < P2) {
            unsigned long long v = (uint32_t)tid < Dt ? dbuf[tid] : ~0ull;
            bar_named(P2);
            switch (P2) {
              case 32: v = bitonic1<5>(v, dbuf, buf0); break;
              case 64: v = bitonic1<6>(v, dbuf, buf0); break;
              case 128: v = bitonic1<7>(v, dbuf, buf0); break;
              case 256: v = bitonic1<8>(v, dbuf, buf0); break;
              default: v = bitonic1<9>(v, dbuf, buf0); break;
            }
            bar_named(P2);
            dbuf[tid] = v;
          }
        } else if (NT == 256) {
          if (P2 == 512) pf_sortE<256, 9>(dbuf, buf0, Dt);
          else pf_sortE<256, 10>(dbuf, buf0, Dt);
        } else {
          pf_sortE<512, 10>(dbuf, buf0, Dt);
        }
      }
      __syncthreads();
      {   // this thread's kept words are consecutive: one search, then a walk
        uint32_t r = 0;
        const uint32_t nk = (uint32_t)__popc(keepm);
        for (uint32_t q = 0; q < nk; ++q) {
          const uint32_t i = kofs0 + q;
          const unsigned long long w = buf1[i];
          if (q == 0) r = lower_rank(dbuf, Dt, w);
          else while (r < Dt && dbuf[r] < w) ++r;
          buf0[i + r] = w;
        }
      }
      for (uint32_t j = tid; j < Dt; j += NT) {
        const unsigned long long w = dbuf[j];
        buf0[j + lower_rank(buf1, Kt, w)] = w;
      }
      for (uint32_t j = nq + tid; j < MP; j += NT) buf0[j] = ~0ull;
#ifdef AUGSCHED_DEBUG
      __syncthreads();   // the merged order must be the strictly increasing one the sort gives
      for (uint32_t j = tid; j + 1 < nq; j += NT)
        if (buf0[j] >= buf0[j + 1]) atomicOr(S.err, 8u);
#endif
      inc_ok = true;
#ifdef AUGSCHED_FM_TIMING
      if (tid == 0) { atomicAdd(&g_fm_t[9], 1ull); atomicAdd(&g_fm_t[10], (unsigned long long)Dt); }
#endif
    }
    __syncthreads();
  }
  // ---- LSD radix sort of bits [30, 64) (tier:2 | key:32), stable.
  // Counters are warp-major (wcnt[w * NBMAX + d]: the leaders of one warp hit
  // distinct banks unless their digits agree mod 32); thread t owns digits
  // [t * DPT, t * DPT + DPT) for the scan in (digit, warp) order.
  unsigned long long* src = buf0;
  unsigned long long* dst = buf1;
#pragma unroll 1
  for (int p = 0; p < (inc_ok ? 0 : 4); ++p) {
    const int shift = PK_KEY + (p == 0 ? 0 : p == 1 ? 9 : p == 2 ? 18 : 26), bits = p < 2 ? 9 : 8;
    const int NB = 1 << bits;
    for (int i = tid; i < NBMAX * NW; i += NT) wcnt[i] = 0;
    __syncthreads();
    unsigned long long xv[E];
    uint32_t rk[E];
    int dg[E];
    const uint32_t seg = (uint32_t)warp * 32 * E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      xv[e] = src[seg + e * 32 + lane];
      dg[e] = (int)((xv[e] >> shift) & (unsigned long long)(NB - 1));
    }
    uint16_t* wc = wcnt + warp * NBMAX;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      unsigned peers;
#if AUGSCHED_FM_MATCH
      peers = __match_any_sync(FULL, dg[e]);
#else
      if (bits == 9) peers = digit_peers_full<9>((uint32_t)dg[e]);
      else peers = digit_peers_full<8>((uint32_t)dg[e]);
#endif
      rk[e] = wc[dg[e]] + __popc(peers & lt);
      __syncwarp();
      if (lane == __ffs(peers) - 1) wc[dg[e]] = (uint16_t)(wc[dg[e]] + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    {
      const int DPT = NB / NT > 0 ? NB / NT : 1;   // 2 or 1 (NT = 256), 1 (NT = 512)
      const int d0 = tid * DPT;
      uint32_t sum = 0;
      if (d0 < NB)
        for (int j = 0; j < DPT; ++j)
#pragma unroll
          for (int w = 0; w < NW; ++w) sum += wcnt[w * NBMAX + d0 + j];
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) tsum[warp] = inc;
      __syncthreads();
      uint32_t run = inc - sum;
      for (int w = 0; w < warp; ++w) run += tsum[w];
      if (d0 < NB)
        for (int j = 0; j < DPT; ++j)
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint32_t c = wcnt[w * NBMAX + d0 + j];
            wcnt[w * NBMAX + d0 + j] = (uint16_t)run;
            run += c;
          }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) dst[wc[dg[e]] + rk[e]] = xv[e];
    __syncthreads();
    unsigned long long* t = src; src = dst; dst = t;
  }
  FMT(1);
  // ---- admission (R17), resolution (R20), grant accounting over the order
  const uint32_t c0 = tc_s[0], c1 = tc_s[1], c2 = tc_s[2];
  const uint32_t n = c0 + c1 + c2;
  const long long B = B_s;
  const uint32_t target = pf_target(B, n);
  const uint32_t prev = S.gdirty[inst];
  if (mord) {   // this order is the next step's starting point
    for (uint32_t j = tid; j < n; j += NT) mord[base + j] = (uint32_t)src[j] & SLOT_MASK;
    if (tid == 0) mord_n[inst] = n;
  }
  FMT(2);
  pf_finish<NT, 8, true>(S, cfg, cap, now, inst, base, src, src, dst, n, target, B, order, keyout, grant,
                         admitted, gslot, sel, wsum, freed, nullptr, 0, n);
  __syncthreads();
  FMT(3);
  // ---- the rest of the order; zero grants beyond the prefix (R16)
  const uint32_t adm = admitted[inst];   // written by thread 0 at the end of pf_finish
  for (uint32_t j = adm + tid; j < n; j += NT) {
    const unsigned long long w = src[j];
    order[base + j] = (uint32_t)w & SLOT_MASK;
    keyout[base + j] = (uint32_t)(w >> PK_KEY);
  }
  for (uint32_t j = adm + tid; j < prev && j < MA; j += NT) grant[base + j] = 0;
  __syncthreads();
  FMT(4);
  if (tid == 0) {
    S.gdirty[inst] = adm;
    n_active[inst] = n;
    tier_off[3 * inst] = 0;
    tier_off[3 * inst + 1] = c0;
    tier_off[3 * inst + 2] = c0 + c1;
  }
}

// ====================================================================== full step, one instance
// augsched_step on a single-instance handle: ONE cooperative kernel (one
// 1,024-thread CTA per SM, a contiguous chunk of slots per CTA) runs the
// keys, a stable LSD radix sort of the 34-bit (tier, key) field in four
// passes (9, 9, 8, 8 bits) and the admission, with grid barriers between
// the phases instead of kernel boundaries and no decoupled look-back:
//   K    packed word of every slot of the chunk (Eq.26 key; tier 3 = not
//        queued) -> kA, and the chunk's digit histogram of pass 0
//   per pass p: publish the chunk histogram H[p][cta][digit]; barrier; each
//        CTA sums the published histograms (all CTAs: digit totals; CTAs
//        before it: its own base per digit); then ranks its chunk stably in
//        sub-tiles of 8,192 words (ballot digit peers, warp-private 16-bit
//        counters, a scan over (digit, warp)) and scatters; barrier; the
//        histogram of the next pass over its chunk of the output
//   last pass writes order (slot) and key of every position and the packed
//        words of the first PF_SCAP positions; the tier counts come from
//        its digit totals (the digit's top two bits are the tier)
//   F    CTA 0: admission (R17), resolution (R20), grant accounting over the
//        first min(B, n) words (pf_finish), grants beyond the prefix zeroed.
constexpr int CNT = 1024;          // threads per CTA
constexpr int CEPT = 8;            // words per thread per sub-tile
constexpr int CNW = CNT / 32;
constexpr int CNB = 512;           // widest digit (9 bits)
constexpr uint32_t CSUB = CNT * CEPT;

struct CoopArgs {
  Slots S;
  augsched_config cfg;
  int64_t cap;
  uint64_t now;
  uint32_t N;
  uint32_t max_limit;                // largest token limit (bounds the admitted prefix)
  unsigned long long *kA, *kB;       // [N] packed words (ping-pong)
  unsigned long long* kpre;          // [PF_SCAP] words of the first positions of the order
  uint32_t* hist;                    // [4][G][CNB] per-CTA digit histograms
  uint32_t* tot;                     // [4][CNB] digit totals
  unsigned long long* bar;           // grid-barrier counter (monotone across calls)
  unsigned long long bar_base;       // its value at this call's start
  long long* budget;
  uint32_t *n_active, *tier_off, *order, *keyout, *grant, *admitted, *gslot;
  // time-invariant keys (reading B12): the previous order's words and the
  // output of this one; ti_try: merge the changed slots into tiw_in.
  // vi: the same for R3 / FCFS keys (words recomputed, order checked)
  int ti, ti_try, vi;
  const unsigned long long* tiw_in;
  unsigned long long *tiw_out, *ubuf;
  const uint32_t* ti_n_in;
  uint32_t* ti_n_out;
  uint32_t* ti_misc;
  uint32_t* gcnt;                    // [TI_DCAP + 1] unchanged words per D rank (kept zero between steps)
  // sharded single queue (f4): the limit from the global ledger and, instead
  // of the admission, this shard's offer
  const long long* ledger;           // [2] global (A, P) or null
  unsigned char* offer;              // ShardOffer buffer or null
  uint32_t ocap;
};

// Offer of one shard (augsched_shard_offer): header, the first min(B, n)
// entries of its order, its queued slots holding KV, its Preserve-paused
// slots (local slot ids; the commit adds the rank's base).
struct ShardHdr { uint32_t n_offer, n_local, n_hq, n_hp, overflow, pad[3]; long long A, P; };
struct OfferRec { unsigned long long w; uint32_t dem, kv; };
constexpr uint32_t SH_HCAP = 8192;   // holders of each kind per shard
__host__ __device__ __forceinline__ size_t shard_offer_bytes(uint32_t ocap) {
  return sizeof(ShardHdr) + sizeof(OfferRec) * ((size_t)ocap + 2 * SH_HCAP);
}
__device__ __forceinline__ ShardHdr* sh_hdr(unsigned char* b) { return reinterpret_cast<ShardHdr*>(b); }
__device__ __forceinline__ OfferRec* sh_off(unsigned char* b) { return reinterpret_cast<OfferRec*>(b + sizeof(ShardHdr)); }
__device__ __forceinline__ OfferRec* sh_hq(unsigned char* b, uint32_t ocap) { return sh_off(b) + ocap; }
__device__ __forceinline__ OfferRec* sh_hp(unsigned char* b, uint32_t ocap) { return sh_off(b) + ocap + SH_HCAP; }

// Offer mode, CTA 0 after the order is complete: the first min(n, ocap)
// words with their demand and KV (ocap >= every limit, so this holds the
// shard's first min(B, n) entries for the global B the commit computes),
// and the shard's ledger after its records.
__device__ void pack_offer(const CoopArgs& a, const unsigned long long* words, uint32_t n, long long B) {
  (void)B;
  const Slots& S = a.S;
  const uint32_t m = n < a.ocap ? n : a.ocap;
  OfferRec* o = sh_off(a.offer);
  for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
    const unsigned long long w = __ldcg(&words[j]);
    const uint32_t x = (uint32_t)w & SLOT_MASK;
    o[j] = OfferRec{w, demand_of(S.ctx[x], S.kv[x], S.cpu[x], S.pend[x], a.cfg.s_in), (uint32_t)S.kv[x]};
  }
  if (threadIdx.x == 0) {
    ShardHdr* h = sh_hdr(a.offer);
    h->n_offer = m;
    h->n_local = n;
    h->A = ld_ll(&S.A[0]);
    h->P = ld_ll(&S.P[0]);
  }
}

#ifdef AUGSCHED_COOP_TIMING
__device__ unsigned long long g_coop_arr[16];   // latest arrival per barrier (ns)
#endif
#ifndef AUGSCHED_COOP_CG
#define AUGSCHED_COOP_CG 1   // grid barrier: cooperative_groups grid sync (0: own counter + nanosleep spin)
#endif
__device__ __forceinline__ void coop_barrier(const CoopArgs& a, uint32_t& k) {
  ++k;
#ifdef AUGSCHED_COOP_TIMING
  if (threadIdx.x == 0) atomicMax(&g_coop_arr[k], gtime());
#endif
#if AUGSCHED_COOP_CG
  cooperative_groups::this_grid().sync();
#else
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(a.bar, 1ull);
    const unsigned long long target = a.bar_base + (unsigned long long)k * gridDim.x;
    while (*(volatile unsigned long long*)a.bar < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
#endif
}

#ifdef AUGSCHED_COOP_TIMING
#define CT(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) ct[i] = gtime(); } while (0)
#else
#define CT(i) do {} while (0)
#endif

__device__ __forceinline__ int coop_shift(int p) { return PK_KEY + (p == 0 ? 0 : p == 1 ? 9 : p == 2 ? 18 : 26); }
__device__ __forceinline__ int coop_bits(int p) { return p < 2 ? 9 : 8; }


// ---- time-invariant keys: the incremental full order (reading B12, f1) ----
// Every word of a slot that did not change since the previous step is the
// word it had then, so the previous order minus the changed slots (U) is
// still sorted.  The changed slots' current words (D, <= TI_DCAP, sorted in
// one CTA) are merged in: a U word at compacted index u lands at
// u + |{d in D : d < w}| (a binary search in shared memory), a D word at
// index j at j + |{u in U : u < D[j]}| (U words counted by their rank in D;
// words are unique).  Three grid barriers, then CTA 0 admits over the first
// min(B, n) positions as in the full path.
__device__ __forceinline__ uint32_t lower_bound_sm(const unsigned long long* v, uint32_t n, unsigned long long x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// vi (R3 / FCFS keys): every key moves with time, so an unchanged slot's
// word is read from kA (this step's words by slot, written by the caller's
// K phase) and the unchanged words, taken in the previous order, must still
// be strictly increasing; each CTA checks its chunk, then every CTA checks
// the chunk boundaries.  When they are not (fp32 rounding re-ordered two
// waiting requests), it returns false before writing any output and the
// caller sorts.  Under R3 every waiting score moves by the same alpha*T per
// step, so this is rare.
template <bool vi>
__device__ bool ti_incremental(const CoopArgs& a, unsigned long long* sbuf, unsigned long long* xch, SelShm& sel,
                               unsigned long long* wsum, unsigned long long& freed, long long& B_s, uint32_t& nbar) {
  __shared__ uint32_t cnt_s[4], dn_s, base_s2, nu_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const Slots& S = a.S;
  const Coef k = S.coef[0];
  const augsched_instance_params ip = S.ip[0];
  const uint32_t E = S.ti_ep;
  const uint32_t nprev = __ldcg(a.ti_n_in);
  // CTA 0 builds D while CTAs 1 .. G-1 take the previous order in chunks
  const uint32_t GU = G - 1, cu = c - 1;
  const uint32_t chunk = ((nprev + GU - 1) / GU + 31) & ~31u;
  const uint32_t c0 = c == 0 ? 0u : (cu * chunk < nprev ? cu * chunk : nprev);
  const uint32_t c1 = c == 0 ? 0u : (c0 + chunk < nprev ? c0 + chunk : nprev);
  // a chunk of <= 8 words per thread stays in registers from A to B
  // (element c0 + warp * 256 + e * 32 + lane, e < 8)
  constexpr int TE = 8;
  const bool reg = c1 - c0 <= (uint32_t)CNT * TE;
  // vi checks the order on chunks held in registers (the host enables it
  // only for queues whose chunks fit; a looping chunk falls back here)
  if (vi && chunk > (uint32_t)CNT * TE) return false;
  unsigned long long rw[TE];
  unsigned rb[TE];          // per e: the warp's ballot of unchanged words
  uint32_t* pub = a.hist;   // [G][4]: kept words, their tiers 0..2, (vi) chunk out of order
  // vi: [G][2] first and last unchanged word of each chunk
  unsigned long long* pv = reinterpret_cast<unsigned long long*>(a.hist + ((4 * G + 1) & ~1u));
  __shared__ unsigned long long vfl[2 * CNW];   // vi: per warp first / last unchanged word
  __shared__ uint32_t vbad;
#ifdef AUGSCHED_COOP_TIMING
#ifndef TT_CTA
#define TT_CTA 0
#endif
  unsigned long long tt[8];
#define TT(i) do { if (c == TT_CTA && tid == 0) tt[i] = gtime(); } while (0)
#else
#define TT(i) do {} while (0)
#endif
  TT(0);
  // ---- A: count the unchanged words of the chunk (and their tiers); CTA 0
  // builds D (the changed slots' current words, queued ones only), sorted
  if (tid < 4) cnt_s[tid] = 0;
  if (tid == 0) { dn_s = 0; vbad = 0; }
  __syncthreads();
  {
    uint32_t kc = 0, t0 = 0, t1 = 0;
    if (reg) {
      const uint32_t seg = c0 + (uint32_t)warp * 32 * TE;
      uint32_t dm[TE];
#pragma unroll
      for (int e = 0; e < TE; ++e) {
        const uint32_t i = seg + e * 32 + lane;
        rw[e] = i < c1 ? __ldcg(&a.tiw_in[i]) : 0ull;
      }
#pragma unroll
      for (int e = 0; e < TE; ++e) {
        const uint32_t i = seg + e * 32 + lane;
        dm[e] = i < c1 ? __ldcg(&S.dmark[(uint32_t)rw[e] & SLOT_MASK]) : E;
      }
      if (vi) {   // this step's word of every unchanged slot
#pragma unroll
        for (int e = 0; e < TE; ++e)
          if (dm[e] != E) rw[e] = __ldcg(&a.kA[(uint32_t)rw[e] & SLOT_MASK]);
      }
      unsigned long long prev = 0, first = ~0ull;   // vi: last unchanged word so far in this warp's segment
      bool bad = false;
#pragma unroll
      for (int e = 0; e < TE; ++e) {
        const bool keep = dm[e] != E;
        rb[e] = __ballot_sync(FULL, keep);
        if (keep) {
          ++kc;
          const uint32_t t = (uint32_t)(rw[e] >> PK_TIER);
          t0 += t == 0; t1 += t == 1;
        }
        if (vi && rb[e]) {
          // the unchanged word before each one in order: the nearest lower
          // unchanged lane, else the previous rounds' last
          const unsigned below = rb[e] & ((1u << lane) - 1);
          const int src = below ? 31 - __clz(below) : lane;
          const unsigned long long pw = __shfl_sync(FULL, rw[e], src);
          if (keep) bad |= (below ? pw : prev) >= rw[e] && (below || prev != 0);
          const int lastl = 31 - __clz(rb[e]), firstl = __ffs(rb[e]) - 1;
          if (first == ~0ull) first = __shfl_sync(FULL, rw[e], firstl);
          prev = __shfl_sync(FULL, rw[e], lastl);
        }
      }
      if (vi) {
        if (__any_sync(FULL, bad) && lane == 0) vbad = 1;
        if (lane == 0) { vfl[2 * warp] = first; vfl[2 * warp + 1] = prev; }
      }
    } else {
      for (uint32_t i = c0 + tid; i < c1; i += CNT) {
        const unsigned long long w = __ldcg(&a.tiw_in[i]);
        if (__ldcg(&S.dmark[(uint32_t)w & SLOT_MASK]) != E) {
          ++kc;
          const uint32_t t = (uint32_t)(w >> PK_TIER);
          t0 += t == 0; t1 += t == 1;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kc += __shfl_xor_sync(FULL, kc, o); t0 += __shfl_xor_sync(FULL, t0, o); t1 += __shfl_xor_sync(FULL, t1, o);
    }
    if (lane == 0) { atomicAdd(&cnt_s[0], kc); atomicAdd(&cnt_s[1], t0); atomicAdd(&cnt_s[2], t1); }
  }
  if (c == 0) {
    if (tid == 0) {
      B_s = a.ledger ? token_limit(a.cfg, k, ip, a.cap, ld_ll(&a.ledger[0]), ld_ll(&a.ledger[1]))
                     : token_limit(a.cfg, k, ip, a.cap, ld_ll(&S.A[0]), ld_ll(&S.P[0]));
      a.budget[0] = B_s;
    }
    const uint32_t dc = __ldcg(&S.dcnt[E & 1]);
    for (uint32_t j = tid; j < dc; j += CNT) {
      const uint32_t g = __ldcg(&S.dlist[(E & 1) * TI_DCAP + j]);
      const unsigned long long w = slot_word(k, ip, S.st[g], S.V[g], S.last[g], a.now, g);
      if ((w >> PK_TIER) < 3) sbuf[atomicAdd(&dn_s, 1u)] = w;
    }
    __syncthreads();
    const uint32_t nd = dn_s;
    uint32_t P2 = 32;
    while (P2 < nd) P2 <<= 1;
    if (P2 <= 1024u) {
      if ((uint32_t)tid < P2) {
        unsigned long long v = (uint32_t)tid < nd ? sbuf[tid] : ~0ull;
        bar_named(P2);
        switch (P2) {
          case 32: v = bitonic1<5>(v, sbuf, xch); break;
          case 64: v = bitonic1<6>(v, sbuf, xch); break;
          case 128: v = bitonic1<7>(v, sbuf, xch); break;
          case 256: v = bitonic1<8>(v, sbuf, xch); break;
          case 512: v = bitonic1<9>(v, sbuf, xch); break;
          default: v = bitonic1<10>(v, sbuf, xch); break;
        }
        bar_named(P2);
        sbuf[tid] = v;
      }
    } else if (P2 == 2048) pf_sortE<CNT, 11>(sbuf, xch, nd);
    else if (P2 == 4096) pf_sortE<CNT, 12>(sbuf, xch, nd);
    else pf_sortE<CNT, 13>(sbuf, xch, nd);
    __syncthreads();
    uint32_t dt0 = 0, dt1 = 0;
    for (uint32_t j = tid; j < nd; j += CNT) {
      a.kB[j] = sbuf[j];
      const uint32_t t = (uint32_t)(sbuf[j] >> PK_TIER);
      dt0 += t == 0; dt1 += t == 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { dt0 += __shfl_xor_sync(FULL, dt0, o); dt1 += __shfl_xor_sync(FULL, dt1, o); }
    __shared__ uint32_t dts[2];
    if (tid == 0) { dts[0] = 0; dts[1] = 0; }
    __syncthreads();
    if (lane == 0) { atomicAdd(&dts[0], dt0); atomicAdd(&dts[1], dt1); }
    __syncthreads();
    if (tid == 0) { a.ti_misc[0] = nd; a.ti_misc[1] = dts[0]; a.ti_misc[2] = dts[1]; }
  }
  __syncthreads();
  if (tid < 3) pub[c * 4 + tid] = cnt_s[tid];
  if (vi && tid == 0) {   // the chunk's warps in order: increasing across warp boundaries too
    unsigned long long f = ~0ull, l = 0;
    uint32_t bad = vbad;
    for (int w2 = 0; w2 < CNW; ++w2) {
      const unsigned long long wf = vfl[2 * w2], wl = vfl[2 * w2 + 1];
      if (wf == ~0ull) continue;
      if (l != 0 && wf <= l) bad = 1;
      if (f == ~0ull) f = wf;
      l = wl;
    }
    if (c == 0) { f = ~0ull; l = 0; }   // CTA 0 takes no chunk (it builds D)
    pub[c * 4 + 3] = bad;
    pv[2 * c] = f;
    pv[2 * c + 1] = l;
  }
  TT(1);
  coop_barrier(a, nbar);
  TT(2);
  if (vi) {
    // every CTA: the chunks' unchanged words must increase across chunks
    __shared__ int vok;
    if (tid < 32) {
      unsigned long long f[8], l[8];
      uint32_t bad = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t cc = lane * 8 + q;
        f[q] = ~0ull; l[q] = 0;
        if (cc < G) { f[q] = __ldcg(&pv[2 * cc]); l[q] = __ldcg(&pv[2 * cc + 1]); bad |= __ldcg(&pub[cc * 4 + 3]); }
      }
      unsigned long long lf = ~0ull, ll = 0;   // this lane's 8 chunks, in order
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (f[q] == ~0ull) continue;
        if (ll != 0 && f[q] <= ll) bad = 1;
        if (lf == ~0ull) lf = f[q];
        ll = l[q];
      }
      // the last word of the lanes before this one (words increase if all is well: a max scan)
      unsigned long long m = ll;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, m, o);
        if (lane >= o && y > m) m = y;
      }
      unsigned long long ex = __shfl_up_sync(FULL, m, 1);
      if (lane == 0) ex = 0;
      if (lf != ~0ull && ex != 0 && lf <= ex) bad = 1;
      const bool any_bad = __any_sync(FULL, bad != 0);
      if (lane == 0) vok = any_bad ? 0 : 1;
    }
    __syncthreads();
    if (!vok) return false;   // uniform: every CTA read the same summaries
  }
  // ---- B: compact the unchanged words (stable) into ubuf and place them
  const uint32_t nd = __ldcg(&a.ti_misc[0]);
  for (uint32_t j = tid; j < nd; j += CNT) sbuf[j] = __ldcg(&a.kB[j]);
  if (tid < 32) {
    uint32_t bsum = 0, tsum = 0;
    uint32_t v[8];   // G <= 256: every load in flight at once
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t cc = lane + 32 * q;
      v[q] = cc < G ? __ldcg(&pub[cc * 4]) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tsum += v[q];
      if (lane + 32 * q < c) bsum += v[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { bsum += __shfl_xor_sync(FULL, bsum, o); tsum += __shfl_xor_sync(FULL, tsum, o); }
    if (lane == 0) { base_s2 = bsum; nu_s = tsum; }
  }
  __syncthreads();
  uint32_t* lh = reinterpret_cast<uint32_t*>(xch);   // this CTA's unchanged words per D rank
  for (uint32_t j = tid; j <= nd; j += CNT) lh[j] = 0;
  if (reg && c1 > c0) {
    // warp totals -> the warp's first compacted index
    uint32_t wt = 0;
#pragma unroll
    for (int e = 0; e < TE; ++e) wt += __popc(rb[e]);
    if (lane == 0) wsum[warp] = wt;
    __syncthreads();
    uint32_t u = base_s2;
    for (int w2 = 0; w2 < warp; ++w2) u += (uint32_t)wsum[w2];
    const uint32_t seg = c0 + (uint32_t)warp * 32 * TE;
#pragma unroll
    for (int e = 0; e < TE; ++e) {
      const bool keep = (rb[e] >> lane) & 1u;
      const uint32_t i = seg + e * 32 + lane;
      uint32_t l = 0xFFFFFFFFu;
      if (keep) {
        const unsigned long long w = rw[e];
        l = lower_bound_sm(sbuf, nd, w);
        const uint32_t pos = u + __popc(rb[e] & ((1u << lane) - 1)) + l;
        const uint32_t x = (uint32_t)w & SLOT_MASK;
        a.tiw_out[pos] = w;
        a.order[pos] = x;
        a.keyout[pos] = (uint32_t)(w >> PK_KEY);
        if (pos < a.max_limit) {
          prefetch_l2(&S.ctx[x]); prefetch_l2(&S.kv[x]); prefetch_l2(&S.cpu[x]); prefetch_l2(&S.pend[x]);
        }
      }
      (void)i;
      if (nd > 0) {
        const unsigned peers = __match_any_sync(FULL, l);
        if (keep && lane == __ffs(peers) - 1) atomicAdd(&lh[l], (unsigned)__popc(peers));
      }
      u += __popc(rb[e]);
    }
  } else {
    uint32_t run = base_s2;
    for (uint32_t b0 = c0; b0 < c1; b0 += CNT) {     // block-uniform trip count
      const uint32_t i = b0 + tid;
      unsigned long long w = 0;
      bool keep = false;
      if (i < c1) {
        w = __ldcg(&a.tiw_in[i]);
        keep = __ldcg(&S.dmark[(uint32_t)w & SLOT_MASK]) != E;
      }
      const unsigned bal = __ballot_sync(FULL, keep);
      if (lane == 0) wsum[warp] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, tile = 0;
      for (int w2 = 0; w2 < CNW; ++w2) { const uint32_t x = (uint32_t)wsum[w2]; before += w2 < warp ? x : 0u; tile += x; }
      uint32_t l = 0xFFFFFFFFu;
      if (keep) {
        const uint32_t u = run + before + __popc(bal & ((1u << lane) - 1));
        l = lower_bound_sm(sbuf, nd, w);
        const uint32_t pos = u + l;
        const uint32_t x = (uint32_t)w & SLOT_MASK;
        a.tiw_out[pos] = w;
        a.order[pos] = x;
        a.keyout[pos] = (uint32_t)(w >> PK_KEY);
        if (pos < a.max_limit) {
          prefetch_l2(&S.ctx[x]); prefetch_l2(&S.kv[x]); prefetch_l2(&S.cpu[x]); prefetch_l2(&S.pend[x]);
        }
      }
      // how many unchanged words fall below each D word: count them by
      // their D rank l (a word is below D[j] iff l <= j); the ranks of a
      // chunk's words are few and sorted, so one atomic per distinct rank
      // and warp
      if (nd > 0) {
        const unsigned peers = __match_any_sync(FULL, l);
        if (keep && lane == __ffs(peers) - 1) atomicAdd(&lh[l], (unsigned)__popc(peers));
      }
      run += tile;
      __syncthreads();
    }
  }
  // the CTA's counts per D rank to the global ones (a chunk's words are a
  // narrow key range: few nonzero ranks)
  __syncthreads();
  if (nd > 0)
    for (uint32_t j = tid; j <= nd; j += CNT)
      if (lh[j]) atomicAdd(&a.gcnt[j], lh[j]);
  TT(3);
  coop_barrier(a, nbar);
  TT(4);
  // ---- C: place the changed words (D[j] lands at j + the unchanged words
  // with rank <= j: an inclusive scan of the rank counts); queue size and
  // tier starts
  const uint32_t nu = nu_s;
  if (c * CNT < nd) {
    uint32_t* cs = reinterpret_cast<uint32_t*>(xch);   // inclusive scan of gcnt[0 .. nd)
    constexpr int PER = TI_DCAP / CNT;
    uint32_t v[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t j = tid * PER + q;
      v[q] = j < nd ? __ldcg(&a.gcnt[j]) : 0u;
      sum += v[q];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t run = inc - sum;
    for (int w2 = 0; w2 < warp; ++w2) run += (uint32_t)wsum[w2];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      run += v[q];
      cs[tid * PER + q] = run;
    }
    __syncthreads();
  }
  for (uint32_t j = c * CNT + tid; j < nd; j += G * CNT) {
    const unsigned long long w = sbuf[j];
    const uint32_t pos = j + reinterpret_cast<const uint32_t*>(xch)[j];
    const uint32_t x = (uint32_t)w & SLOT_MASK;
    a.tiw_out[pos] = w;
    a.order[pos] = x;
    a.keyout[pos] = (uint32_t)(w >> PK_KEY);
    if (pos < a.max_limit) {
      prefetch_l2(&S.ctx[x]); prefetch_l2(&S.kv[x]); prefetch_l2(&S.cpu[x]); prefetch_l2(&S.pend[x]);
    }
  }
  if (c == 0 && tid < 32) {
    uint32_t u0 = 0, u1 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t cc = lane + 32 * q;
      if (cc < G) { u0 += __ldcg(&pub[cc * 4 + 1]); u1 += __ldcg(&pub[cc * 4 + 2]); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { u0 += __shfl_xor_sync(FULL, u0, o); u1 += __shfl_xor_sync(FULL, u1, o); }
    if (lane == 0) {
      const uint32_t n = nu + nd;
      const uint32_t t0 = u0 + __ldcg(&a.ti_misc[1]), t1 = u1 + __ldcg(&a.ti_misc[2]);
      a.n_active[0] = n;
      *a.ti_n_out = n;
      a.tier_off[0] = 0;
      a.tier_off[1] = t0;
      a.tier_off[2] = t0 + t1;
    }
  }
  TT(5);
  coop_barrier(a, nbar);
  TT(6);
#ifdef AUGSCHED_DEBUG
  {   // the merged order is strictly increasing (checked over each CTA's share)
    const uint32_t nt = nu + nd, per = (nt + G - 1) / G;
    const uint32_t q0 = c * per, q1 = q0 + per < nt ? q0 + per : nt;
    for (uint32_t i = q0 + tid; i < q1; i += CNT)
      if (i + 1 < nt && __ldcg(&a.tiw_out[i]) >= __ldcg(&a.tiw_out[i + 1])) atomicOr(S.err, 8u);
  }
#endif
#ifdef AUGSCHED_COOP_TIMING
  if (c == TT_CTA && c != 0 && tid == 0)
    printf("ti_t cta %u ns: nd %u | %llu %llu %llu %llu %llu %llu\n", c, nd, tt[1] - tt[0], tt[2] - tt[0],
           tt[3] - tt[0], tt[4] - tt[0], tt[5] - tt[0], tt[6] - tt[0]);
#endif
  if (c != 0) return true;
  for (uint32_t j = tid; j <= nd; j += CNT) a.gcnt[j] = 0;   // clear for the next step
  // ---- F: admission over the first min(B, n) positions (CTA 0)
  const uint32_t n = __ldcg(&a.n_active[0]);
  const long long B = B_s;
  if (a.offer) { pack_offer(a, a.tiw_out, n, B); return true; }
  const uint32_t target = pf_target(B, n);
  for (uint32_t i = tid; i < target; i += CNT) sbuf[i] = __ldcg(&a.tiw_out[i]);
  const uint32_t prev = S.gdirty[0];
  __syncthreads();
  pf_finish<CNT, PF_SCAP / CNT, true>(S, a.cfg, a.cap, a.now, 0, 0, nullptr, sbuf, nullptr, target, target, B,
                                      a.order, a.keyout, a.grant, a.admitted, a.gslot, sel, wsum, freed);
  __syncthreads();
  const uint32_t adm = a.admitted[0];
  for (uint32_t j = adm + tid; j < prev && j < a.N; j += CNT) a.grant[j] = 0;
  if (tid == 0) S.gdirty[0] = adm;
#ifdef AUGSCHED_COOP_TIMING
  TT(7);
  if (tid == 0) printf("ti_t ns: nd %u | %llu %llu %llu %llu %llu %llu %llu\n", nd, tt[1] - tt[0], tt[2] - tt[0],
                       tt[3] - tt[0], tt[4] - tt[0], tt[5] - tt[0], tt[6] - tt[0], tt[7] - tt[0]);
#endif
#undef TT
  return true;
}

// VI: the instantiation for value (R3) / FCFS keys (K phase first, then the
// checked merge or the sort); the other one serves time-invariant keys and
// handles without a kept order.
template <bool VI>
__global__ void __launch_bounds__(CNT, 1) full_coop_kernel(const __grid_constant__ CoopArgs a) {
  extern __shared__ __align__(16) unsigned long long fc_sm[];
  unsigned long long* sbuf = fc_sm;                                            // [PF_SCAP] (phase F)
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(fc_sm + PF_SCAP);              // [CNW][CNB]
  __shared__ uint32_t h[CNB];          // chunk histogram of the next pass
  __shared__ uint32_t base_s[CNB];     // running position of each digit for this CTA
  __shared__ uint32_t tot_s[CNB];      // digit totals (all CTAs)
  __shared__ uint32_t wsc[CNW + 1];
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[CNW + 1];
  __shared__ unsigned long long freed;
  __shared__ long long B_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1;
  const uint32_t G = gridDim.x, c = blockIdx.x, N = a.N;
  const Slots& S = a.S;
  const uint32_t chunk = ((N + G - 1) / G + 31) & ~31u;
  const uint32_t c0 = c * chunk < N ? c * chunk : N;
  const uint32_t c1 = c0 + chunk < N ? c0 + chunk : N;
  uint32_t nbar = 0;
  const bool inc = a.ti_try && __ldcg(&S.dcnt[S.ti_ep & 1]) <= TI_DCAP;   // uniform: the list is final at launch
  if (!VI && inc && a.ti) {
    ti_incremental<false>(a, sbuf, reinterpret_cast<unsigned long long*>(wcnt), sel, wsum, freed, B_s, nbar);
    return;
  }
  const bool vi = VI && inc && a.vi;   // R3 / FCFS: the words first (K), then the merge or, failing that, the sort
#ifdef AUGSCHED_COOP_TIMING
  unsigned long long ct[32];
#endif
  CT(0);
  // A chunk that fits one sub-tile stays in registers between the phases
  // (xr, element i = c0 + warp * 256 + e * 32 + lane, the ranking order):
  // the words are not written by K, and each pass's input is read once.
  const bool reg = c1 - c0 <= CSUB && !vi;   // vi gathers this step's words from kA
  unsigned long long xr[CEPT];
  // ---- K: words of the chunk + histogram of pass 0
  {
    const Coef k = S.coef[0];
    const augsched_instance_params ip = S.ip[0];
    for (int b = tid; b < CNB; b += CNT) h[b] = 0;
    __syncthreads();
    for (uint32_t b0 = c0; b0 < c1; b0 += CSUB) {   // block-uniform trip count
      uint32_t stv[CEPT], lst[CEPT];
      double V[CEPT];
      const uint32_t seg = b0 + (uint32_t)warp * 32 * CEPT;
#pragma unroll
      for (int u = 0; u < CEPT; ++u) {
        const uint32_t x = seg + u * 32 + lane;
        stv[u] = 0u; lst[u] = 0u; V[u] = 0.0;
        if (x < c1) { stv[u] = S.st[x]; V[u] = S.V[x]; lst[u] = S.last[x]; }
      }
#pragma unroll
      for (int u = 0; u < CEPT; ++u) {
        const uint32_t x = seg + u * 32 + lane;
        const unsigned long long w = slot_word(k, ip, stv[u], V[u], lst[u], a.now, x);
        xr[u] = w;
        if (x < c1 && !reg) a.kA[x] = w;
        hist_add(h, x < c1 ? (int)((w >> coop_shift(0)) & (CNB - 1)) : -1);
      }
    }
    if (c == 0 && tid == 0) {
      B_s = a.ledger ? token_limit(a.cfg, k, ip, a.cap, ld_ll(&a.ledger[0]), ld_ll(&a.ledger[1]))
                     : token_limit(a.cfg, k, ip, a.cap, ld_ll(&S.A[0]), ld_ll(&S.P[0]));
      a.budget[0] = B_s;
    }
  }
  if (vi) {
    coop_barrier(a, nbar);   // kA complete
    if (ti_incremental<VI>(a, sbuf, reinterpret_cast<unsigned long long*>(wcnt), sel, wsum, freed, B_s, nbar))
      return;
    // out of order: sort (kA and the pass-0 histogram h are intact)
  }
  unsigned long long* src = a.kA;
  unsigned long long* dst = a.kB;
#pragma unroll 1
  for (int p = 0; p < 4; ++p) {
    const int shift = coop_shift(p), bits = coop_bits(p), NB = 1 << bits;
    const bool last = p == 3;
    // publish the chunk histogram of this pass
    __syncthreads();
    uint32_t* Hp = a.hist + (size_t)p * G * CNB;
    for (int b = tid; b < NB; b += CNT) Hp[(size_t)c * CNB + b] = h[b];
    CT(1 + 6 * p);
    coop_barrier(a, nbar);
    CT(2 + 6 * p);
    // column scan: CTA c owns digits [c * DPC, c * DPC + DPC) and scans
    // each over the G CTAs (thread tid: digit j = tid / 256, CTA tid % 256),
    // writing the exclusive prefixes back in place and the digit total
    {
      const int DPC = (NB + (int)G - 1) / (int)G;        // <= 4 (G >= 128)
      const int j = tid >> 8, cc = tid & 255;
      const int d = (int)c * DPC + j;
      const bool own = j < DPC && d < NB && cc < (int)G;
      const uint32_t v = own ? __ldcg(&Hp[(size_t)cc * CNB + d]) : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) wsc[warp] = inc;
      __syncthreads();
      uint32_t run = inc - v;
      for (int w = j * 8; w < warp; ++w) run += wsc[w];   // the 8 warps of digit group j
      if (own) Hp[(size_t)cc * CNB + d] = run;
      if (j < DPC && d < NB && cc == 255) a.tot[p * CNB + d] = run + v;
    }
    coop_barrier(a, nbar);
    // this CTA's base per digit: exclusive scan of the totals over digits
    // plus its own column prefix
    {
      const uint32_t v = tid < NB ? __ldcg(&a.tot[p * CNB + tid]) : 0u;
      const uint32_t pre = tid < NB ? __ldcg(&Hp[(size_t)c * CNB + tid]) : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      __syncthreads();   // wsc reuse
      if (lane == 31) wsc[warp] = inc;
      __syncthreads();
      uint32_t run = inc - v;
      for (int w = 0; w < warp; ++w) run += wsc[w];
      if (tid < NB) { base_s[tid] = run + pre; tot_s[tid] = v; }
      __syncthreads();
    }
    CT(3 + 6 * p);
    if (last && c == 0 && tid == 0) {
      // tier counts: the last digit's top two bits are the tier
      uint32_t tc[4] = {0u, 0u, 0u, 0u};
      for (int d = 0; d < NB; ++d) tc[d >> 6] += tot_s[d];
      const uint32_t n = tc[0] + tc[1] + tc[2];
      a.n_active[0] = n;
      if (a.ti || a.vi) *a.ti_n_out = n;
      a.tier_off[0] = 0;
      a.tier_off[1] = tc[0];
      a.tier_off[2] = tc[0] + tc[1];
    }
    // rank and scatter the chunk, sub-tile by sub-tile
    for (uint32_t s0 = c0; s0 < c1; s0 += CSUB) {
      for (int i = tid; i < CNW * CNB; i += CNT) wcnt[i] = 0;
      __syncthreads();
      unsigned long long xv[CEPT];
      uint32_t rk[CEPT];
      int dg[CEPT];
      const uint32_t seg = s0 + (uint32_t)warp * 32 * CEPT;
#pragma unroll
      for (int e = 0; e < CEPT; ++e) {
        const uint32_t i = seg + e * 32 + lane;
        xv[e] = i >= c1 ? 0ull : reg ? xr[e] : __ldcg(&src[i]);
        dg[e] = i < c1 ? (int)((xv[e] >> shift) & (unsigned long long)(NB - 1)) : -1;
      }
      uint16_t* wc = wcnt + warp * CNB;
#pragma unroll
      for (int e = 0; e < CEPT; ++e) {
        unsigned peers;
        if (bits == 9) peers = digit_peers<9>(dg[e]);
        else peers = digit_peers<8>(dg[e]);
        if (dg[e] >= 0) rk[e] = wc[dg[e]] + __popc(peers & lt);
        __syncwarp();
        if (dg[e] >= 0 && lane == __ffs(peers) - 1) wc[dg[e]] = (uint16_t)(wc[dg[e]] + __popc(peers));
        __syncwarp();
      }
      __syncthreads();
      // per digit: exclusive offsets over the warps, advance the running base
      for (int d = tid; d < NB; d += CNT) {
        uint32_t run = base_s[d];
#pragma unroll 8
        for (int w = 0; w < CNW; ++w) {
          const uint32_t v = wcnt[w * CNB + d];
          wcnt[w * CNB + d] = (uint16_t)(run - base_s[d]);
          run += v;
        }
        tot_s[d] = run;   // the base for the next sub-tile (tot_s is free after the scan)
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < CEPT; ++e) {
        if (dg[e] < 0) continue;
        const uint32_t pos = base_s[dg[e]] + wc[dg[e]] + rk[e];
        if (last) {
          const uint32_t x = (uint32_t)xv[e] & SLOT_MASK;
          a.order[pos] = x;
          a.keyout[pos] = (uint32_t)(xv[e] >> PK_KEY);
          if (pos < PF_SCAP) a.kpre[pos] = xv[e];
          if (a.ti || a.vi) a.tiw_out[pos] = xv[e];   // the order the next step merges into
          if (pos < a.max_limit) {   // the admission (phase F) reads these slots' token state
            prefetch_l2(&S.ctx[x]); prefetch_l2(&S.kv[x]); prefetch_l2(&S.cpu[x]); prefetch_l2(&S.pend[x]);
          }
        } else {
          dst[pos] = xv[e];
        }
      }
      __syncthreads();
      for (int d = tid; d < NB; d += CNT) base_s[d] = tot_s[d];
      __syncthreads();
    }
    CT(4 + 6 * p);
    coop_barrier(a, nbar);
    CT(5 + 6 * p);
    if (!last) {
      // histogram of the next pass over this CTA's chunk of the output
      const int ns = coop_shift(p + 1);
      const int nm = (1 << coop_bits(p + 1)) - 1;
      for (int b = tid; b < CNB; b += CNT) h[b] = 0;
      __syncthreads();
      for (uint32_t i0 = c0; i0 < c1; i0 += CSUB) {
        const uint32_t seg = i0 + (uint32_t)warp * 32 * CEPT;
#pragma unroll
        for (int u = 0; u < CEPT; ++u) {
          const uint32_t i = seg + u * 32 + lane;
          xr[u] = i < c1 ? __ldcg(&dst[i]) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < CEPT; ++u) {
          const uint32_t i = seg + u * 32 + lane;
          hist_add(h, i < c1 ? (int)((xr[u] >> ns) & (unsigned long long)nm) : -1);
        }
      }
      unsigned long long* t = src; src = dst; dst = t;
    }
    CT(6 + 6 * p);
  }
  if (c != 0) return;
  // ---- F: admission over the first min(B, n) positions
  const uint32_t n = __ldcg(&a.n_active[0]);
  const long long B = B_s;
  if (a.offer) { pack_offer(a, a.kpre, n, B); return; }
  const uint32_t target = pf_target(B, n);
  for (uint32_t i = tid; i < target; i += CNT) sbuf[i] = __ldcg(&a.kpre[i]);
  const uint32_t prev = S.gdirty[0];
  __syncthreads();
  pf_finish<CNT, PF_SCAP / CNT, true>(S, a.cfg, a.cap, a.now, 0, 0, nullptr, sbuf, nullptr, target, target, B,
                                      a.order, a.keyout, a.grant, a.admitted, a.gslot, sel, wsum, freed);
  __syncthreads();
  const uint32_t adm = a.admitted[0];
  for (uint32_t j = adm + tid; j < prev && j < N; j += CNT) a.grant[j] = 0;
  if (tid == 0) S.gdirty[0] = adm;
#ifdef AUGSCHED_COOP_TIMING
  CT(25);
  if (tid == 0) {
    printf("coop_t ns:");
    for (int i = 1; i <= 25; ++i) printf(" %llu", ct[i] - ct[0]);
    printf("\ncoop_arr ns:");
    for (int i = 1; i <= 12; ++i) { printf(" %llu", g_coop_arr[i] - ct[0]); g_coop_arr[i] = 0; }
    printf("\n");
  }
#endif
}

// ====================================================================== sharded single queue (f4)
// This shard's KV holders for the global R20 resolution: queued slots with
// kv > 0 (their packed word) and Preserve-paused slots with kv > 0 (their
// demotion key (2^32-1-kv) << 30 | slot: kv desc, slot asc).
__global__ void shard_holders_kernel(Slots S, uint64_t now, uint32_t N, unsigned char* offer, uint32_t ocap) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= N) return;
  const uint32_t stv = S.st[x], s4 = stv & 15;
  const int32_t kv = S.kv[x];
  if (kv <= 0) return;
  ShardHdr* h = sh_hdr(offer);
  if (s4 >= ST_RUN && s4 <= ST_WAIT) {
    const unsigned long long w = slot_word(S.coef[0], S.ip[0], stv, S.V[x], S.last[x], now, x);
    const uint32_t q = atomicAdd(&h->n_hq, 1u);
    if (q < SH_HCAP) sh_hq(offer, ocap)[q] = OfferRec{w, 0u, (uint32_t)kv};
    else atomicOr(&h->overflow, 2u);
  } else if (s4 == ST_PAUSED && ((stv >> 4) & 3) == POL_P) {
    const uint32_t q = atomicAdd(&h->n_hp, 1u);
    const unsigned long long key = ((unsigned long long)(0xFFFFFFFFu - (uint32_t)kv) << 30) | x;
    if (q < SH_HCAP) sh_hp(offer, ocap)[q] = OfferRec{key, 0u, (uint32_t)kv};
    else atomicOr(&h->overflow, 4u);
  }
}

struct CommitArgs {
  Slots S;
  augsched_config cfg;
  int64_t cap;
  uint64_t now;
  const unsigned char* offers;   // n_ranks blocks of shard_offer_bytes(ocap)
  size_t obytes;
  uint32_t ocap, n_ranks, rank, MA;
  long long* gledger;            // [2] global (A, P) after this step (the next step's C_other base)
  long long* budget;
  uint32_t *n_active, *admitted, *order, *keyout, *grant, *err;
};

__device__ __forceinline__ const unsigned char* cm_blk(const CommitArgs& a, uint32_t r) { return a.offers + (size_t)r * a.obytes; }
// global packed word of record j of rank r's list
__device__ __forceinline__ unsigned long long cm_gword(const CommitArgs& a, uint32_t r, unsigned long long w) {
  return (w & ~(unsigned long long)SLOT_MASK) | ((unsigned long long)r * a.MA + ((uint32_t)w & SLOT_MASK));
}
// the offer record of global word gw (it is in its rank's sorted offer list)
__device__ const OfferRec* cm_find(const CommitArgs& a, unsigned long long gw) {
  const uint32_t gs = (uint32_t)gw & SLOT_MASK, r = gs / a.MA;
  const unsigned char* b = cm_blk(a, r);
  const uint32_t n = reinterpret_cast<const ShardHdr*>(b)->n_offer;
  const OfferRec* o = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr));
  const unsigned long long lw = (gw & ~(unsigned long long)SLOT_MASK) | (gs - r * a.MA);
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (o[mid].w < lw) lo = mid + 1; else hi = mid;
  }
  return &o[lo];
}

// One CTA: merge the offers (the target smallest global words by a count
// select, then a bitonic sort), admit the global prefix (R17), resolve
// memory pressure over the gathered holders (R20: demote Preserve-paused by
// kv desc / slot asc, then evict from the tail of the global order over
// entries with kv + g > 0), write the global prefix and apply this shard's
// part.
__global__ void __launch_bounds__(1024, 1) shard_commit_kernel(const __grid_constant__ CommitArgs a) {
  constexpr int NT = 1024;
  extern __shared__ __align__(16) unsigned long long cm_sm[];
  unsigned long long* sbuf = cm_sm;            // [PF_SCAP] the admitted candidates, sorted
  unsigned long long* xch = cm_sm + PF_SCAP;   // [PF_SCAP] sort exchange, then the grants (u32)
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[NT / 32 + 1];
  __shared__ unsigned long long freed_s;
  __shared__ uint32_t m_s, tot_off_s, n_tot_s, ovf_s;
  __shared__ long long B_s;
  const int tid = threadIdx.x;
  const Slots& S = a.S;
  const uint32_t G = a.n_ranks, OC = a.ocap;
  __shared__ long long gA_s, gP_s;
  if (tid == 0) {
    const Coef k = S.coef[0];
    uint32_t to = 0, nt = 0, ov = 0;
    long long A = 0, P = 0;
    for (uint32_t r = 0; r < G; ++r) {
      const ShardHdr* h = reinterpret_cast<const ShardHdr*>(cm_blk(a, r));
      to += h->n_offer; nt += h->n_local; ov |= h->overflow; A += h->A; P += h->P;
    }
    gA_s = A; gP_s = P;
    B_s = token_limit(a.cfg, k, S.ip[0], a.cap, A, P);   // Eq.27-32 on the global ledger
    tot_off_s = to; n_tot_s = nt; ovf_s = ov; m_s = 0;
    a.budget[0] = B_s;
    a.n_active[0] = nt;
  }
  __syncthreads();
  const long long B = B_s;
  const uint32_t target = pf_target(B, tot_off_s);
  auto off_get = [&](uint32_t i, uint64_t& key, uint32_t& w) -> bool {
    const uint32_t r = i / OC, j = i - r * OC;
    const unsigned char* b = cm_blk(a, r);
    if (j >= reinterpret_cast<const ShardHdr*>(b)->n_offer) return false;
    key = cm_gword(a, r, reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr))[j].w);
    w = 1u;
    return true;
  };
  if (target > 0) {
    wselect<NT>(sel, G * OC, target, 64, off_get);
    const unsigned long long tau = sel.r.found ? sel.r.k : ~0ull;
    for (uint32_t i = tid; i < G * OC; i += NT) {
      uint64_t key; uint32_t w;
      if (off_get(i, key, w) && key <= tau) sbuf[atomicAdd(&m_s, 1u)] = key;
    }
    __syncthreads();
    const uint32_t mt = m_s;
    uint32_t P2 = 32;
    while (P2 < mt) P2 <<= 1;
    if (P2 <= 1024u) {
      if ((uint32_t)tid < P2) {
        unsigned long long v = (uint32_t)tid < mt ? sbuf[tid] : ~0ull;
        bar_named(P2);
        switch (P2) {
          case 32: v = bitonic1<5>(v, sbuf, xch); break;
          case 64: v = bitonic1<6>(v, sbuf, xch); break;
          case 128: v = bitonic1<7>(v, sbuf, xch); break;
          case 256: v = bitonic1<8>(v, sbuf, xch); break;
          case 512: v = bitonic1<9>(v, sbuf, xch); break;
          default: v = bitonic1<10>(v, sbuf, xch); break;
        }
        bar_named(P2);
        sbuf[tid] = v;
      }
    } else if (P2 == 2048) pf_sortE<NT, 11>(sbuf, xch, mt);
    else if (P2 == 4096) pf_sortE<NT, 12>(sbuf, xch, mt);
    else pf_sortE<NT, 13>(sbuf, xch, mt);
    __syncthreads();
  }
  uint32_t* gs = reinterpret_cast<uint32_t*>(xch);   // grant of prefix position j
  // ---- a6 admission over the global prefix (P_{j-1} < B, partial last, R17)
  unsigned long long Prun = 0, gsum = 0;
  uint32_t adm = 0;
  for (uint32_t j0 = 0; j0 < target && (long long)Prun < B; j0 += NT) {
    const uint32_t j = j0 + tid;
    unsigned long long d = 0;
    if (j < target) d = cm_find(a, sbuf[j])->dem;
    unsigned long long tot;
    const unsigned long long inc = block_incl_scan_u64<NT>(d, wsum, &tot);
    const unsigned long long ex = Prun + inc - d;
    const bool in = j < target && (long long)ex < B;
    if (j < target) gs[j] = 0;
    if (in) {
      const unsigned long long g = d < (unsigned long long)B - ex ? d : (unsigned long long)B - ex;
      gs[j] = (uint32_t)g;
      gsum += g;
    }
    adm += __syncthreads_count(in);
    Prun += tot;
  }
  unsigned long long need;
  block_incl_scan_u64<NT>(gsum, wsum, &need);
  long long fr = a.cap - gA_s - gP_s;
  // ---- a7 resolution over the gathered holders (rare)
  bool demote = false, evict = false;
  unsigned long long k0 = 0, k1 = 0;
  bool f0 = false, f1 = false;
  auto hp_get = [&](uint32_t i, uint64_t& key, uint32_t& w) -> bool {
    const uint32_t r = i / SH_HCAP, j = i - r * SH_HCAP;
    const unsigned char* b = cm_blk(a, r);
    const uint32_t n = reinterpret_cast<const ShardHdr*>(b)->n_hp;
    if (j >= (n < SH_HCAP ? n : SH_HCAP)) return false;
    const OfferRec rec = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr))[OC + SH_HCAP + j];
    key = (rec.w & ~(unsigned long long)SLOT_MASK) | ((unsigned long long)r * a.MA + ((uint32_t)rec.w & SLOT_MASK));
    w = rec.kv;
    return true;
  };
  // eviction candidates: holders_q (kv + their grant if admitted) and the
  // admitted entries that hold no KV (their grant); key = ~word (tail first)
  auto adm_pos = [&](unsigned long long gw) -> int {
    uint32_t lo = 0, hi = adm;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sbuf[mid] < gw) lo = mid + 1; else hi = mid;
    }
    return lo < adm && sbuf[lo] == gw ? (int)lo : -1;
  };
  auto ev_get = [&](uint32_t i, uint64_t& key, uint32_t& w) -> bool {
    if (i < G * SH_HCAP) {
      const uint32_t r = i / SH_HCAP, j = i - r * SH_HCAP;
      const unsigned char* b = cm_blk(a, r);
      const uint32_t n = reinterpret_cast<const ShardHdr*>(b)->n_hq;
      if (j >= (n < SH_HCAP ? n : SH_HCAP)) return false;
      const OfferRec rec = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr))[OC + j];
      const unsigned long long gw = cm_gword(a, r, rec.w);
      const int p = adm_pos(gw);
      w = rec.kv + (p >= 0 ? gs[p] : 0u);
      key = ~gw;
      return w > 0;
    }
    const uint32_t j = i - G * SH_HCAP;
    if (j >= adm || gs[j] == 0) return false;
    if (cm_find(a, sbuf[j])->kv > 0) return false;   // listed with the holders
    key = ~sbuf[j];
    w = gs[j];
    return true;
  };
  if ((long long)need > fr) {
    if (ovf_s & 6u) { if (tid == 0) atomicOr(a.err, 2u); }   // a shard's holder list overflowed
    demote = true;
    wselect<NT>(sel, G * SH_HCAP, (uint64_t)((long long)need - fr), 62, hp_get);
    f0 = sel.r.found != 0;
    k0 = sel.r.k;
    if (tid == 0) freed_s = 0;
    __syncthreads();
    for (uint32_t i = tid; i < G * SH_HCAP; i += NT) {
      uint64_t key; uint32_t w;
      if (hp_get(i, key, w) && (!f0 || key <= k0)) atomicAdd(&freed_s, (unsigned long long)w);
    }
    __syncthreads();
    fr += (long long)freed_s;
    if (tid == 0) gP_s -= (long long)freed_s;   // demoted KV leaves P
    if ((long long)need > fr) {
      evict = true;
      wselect<NT>(sel, G * SH_HCAP + adm, (uint64_t)((long long)need - fr), 64, ev_get);
      f1 = sel.r.found != 0;
      k1 = sel.r.k;
      __syncthreads();
      // admitted entries that are evicted (their candidate key passes; kv + g > 0
      // holds for them): grant cancelled, marked until this shard applied it
      for (uint32_t j = tid; j < adm; j += NT)
        if (gs[j] > 0 && (!f1 || ~sbuf[j] <= k1)) gs[j] = 0xFFFFFFFFu;
      // KV released by the evicted holders of every shard leaves A
      if (tid == 0) freed_s = 0;
      __syncthreads();
      for (uint32_t i = tid; i < G * SH_HCAP; i += NT) {
        const uint32_t r = i / SH_HCAP, j = i - r * SH_HCAP;
        const unsigned char* b = cm_blk(a, r);
        const uint32_t n = reinterpret_cast<const ShardHdr*>(b)->n_hq;
        if (j >= (n < SH_HCAP ? n : SH_HCAP)) continue;
        const OfferRec rec = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr))[OC + j];
        if (!f1 || ~cm_gword(a, r, rec.w) <= k1) atomicAdd(&freed_s, (unsigned long long)rec.kv);
      }
      __syncthreads();
      if (tid == 0) gA_s -= (long long)freed_s;
    }
  }
  __syncthreads();
  // ---- outputs (every rank the same) and this shard's part
  const uint32_t base = a.rank * a.MA;
  long long dA = 0, dP = 0;
  for (uint32_t j = tid; j < adm; j += NT) {
    const unsigned long long gw = sbuf[j];
    const uint32_t g = gs[j];
    a.order[j] = (uint32_t)gw & SLOT_MASK;
    a.keyout[j] = (uint32_t)(gw >> PK_KEY);
    a.grant[j] = g == 0xFFFFFFFFu ? 0u : g;
    const uint32_t gsl = (uint32_t)gw & SLOT_MASK;
    if (g == 0xFFFFFFFFu && gsl >= base && gsl < base + a.MA) {
      // this shard's evicted admitted entry: whole context recomputed (B2);
      // its KV (if any) is released by the holder loop below
      const uint32_t x = gsl - base;
      S.cpu[x] = 0;
      S.st[x] = ST_WAIT | (S.st[x] & 0x30u);
      mark_dirty(S, x, S.ti_ep + 1);
    }
  }
  if (evict) {   // this shard's evicted holders (queued, kv > 0) and admitted KV-free entries
    const unsigned char* b = cm_blk(a, a.rank);
    const uint32_t nq = reinterpret_cast<const ShardHdr*>(b)->n_hq;
    const OfferRec* hq = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr)) + OC;
    for (uint32_t j = tid; j < (nq < SH_HCAP ? nq : SH_HCAP); j += NT) {
      const unsigned long long gw = cm_gword(a, a.rank, hq[j].w);
      if (!f1 || ~gw <= k1) {
        const uint32_t x = (uint32_t)hq[j].w & SLOT_MASK;
        dA -= S.kv[x];
        S.kv[x] = 0; S.cpu[x] = 0;
        S.st[x] = ST_WAIT | (S.st[x] & 0x30u);
        mark_dirty(S, x, S.ti_ep + 1);
      }
    }
  }
  if (demote) {
    const unsigned char* b = cm_blk(a, a.rank);
    const uint32_t np = reinterpret_cast<const ShardHdr*>(b)->n_hp;
    const OfferRec* hp = reinterpret_cast<const OfferRec*>(b + sizeof(ShardHdr)) + OC + SH_HCAP;
    for (uint32_t j = tid; j < (np < SH_HCAP ? np : SH_HCAP); j += NT) {
      const uint32_t x = (uint32_t)hp[j].w & SLOT_MASK;
      const unsigned long long key = (hp[j].w & ~(unsigned long long)SLOT_MASK) | (base + x);
      if (!f0 || key <= k0) {
        dP -= S.kv[x];
        S.kv[x] = 0;
        S.st[x] = ST_PAUSED | ((uint32_t)POL_D << 4);
      }
    }
  }
  __syncthreads();
  for (uint32_t j = tid; j < adm; j += NT) {
    const uint32_t gsl = (uint32_t)sbuf[j] & SLOT_MASK;
    const uint32_t gr = gs[j];
    if (gsl < base || gsl >= base + a.MA || gr == 0 || gr == 0xFFFFFFFFu) continue;
    const uint32_t x = gsl - base;
    int32_t ctx = S.ctx[x], kv = S.kv[x], cpu = S.cpu[x], pend = S.pend[x];
    if (cpu > 0) { cpu -= (int32_t)gr; kv += (int32_t)gr; }
    else if ((ctx - kv) + pend > 0) {
      const int32_t rc = (int32_t)gr < ctx - kv ? (int32_t)gr : ctx - kv;
      kv += rc;
      const int32_t pp = (int32_t)gr - rc;
      pend -= pp; ctx += pp; kv += pp;
    } else { ctx += 1; kv += 1; }
    dA += gr;
    S.ctx[x] = ctx; S.kv[x] = kv; S.cpu[x] = cpu; S.pend[x] = pend;
    S.last[x] = (uint32_t)a.now;
    S.st[x] = ST_RUN | (S.st[x] & 0x30u);
    mark_dirty(S, x, S.ti_ep + 1);
  }
  // tokens granted over all shards (every admitted grant that stands)
  unsigned long long gt = 0;
  for (uint32_t j = tid; j < adm; j += NT) gt += gs[j] == 0xFFFFFFFFu ? 0u : gs[j];
  unsigned long long tA, tP, tG;
  block_incl_scan_u64<NT>((unsigned long long)dA, wsum, &tA);
  block_incl_scan_u64<NT>((unsigned long long)dP, wsum, &tP);
  block_incl_scan_u64<NT>(gt, wsum, &tG);
  if (tid == 0) {
    a.gledger[0] = gA_s + (long long)tG;
    a.gledger[1] = gP_s;
    a.admitted[0] = adm;
    const long long A = ld_ll(&S.A[0]) + (long long)tA;
    S.A[0] = A;
    S.Aevt[0] = A;
    S.P[0] = ld_ll(&S.P[0]) + (long long)tP;
  }
}
}  // namespace

// ====================================================================== host
namespace {

template <class T>
int salloc(StepState& st, T** p, size_t n) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(e == cudaErrorMemoryAllocation ? AUGSCHED_E_OOM : AUGSCHED_E_CUDA,
                     "step: device allocation failed");
  }
  st.alloc_list[st.n_alloc++] = *p;
  return AUGSCHED_OK;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return AUGSCHED_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  return set_error(AUGSCHED_E_CUDA, buf);
}

int grow_records(StepState& st, uint32_t need, cudaStream_t s) {
  if (need <= st.r_cap) return AUGSCHED_OK;
  uint32_t cap = st.r_cap ? st.r_cap : 1024;
  while (cap < need) cap *= 2;
  uint32_t** u[] = {&st.r_kind, &st.r_id, &st.r_la, &st.r_lb, &st.r_lc, &st.r_flags, &st.r_last,
                    &st.r_ctx, &st.r_kv, &st.r_cpu, &st.r_pend};
  for (auto pp : u) {
    uint32_t* np = nullptr;
    if (cudaMalloc(&np, sizeof(uint32_t) * cap) != cudaSuccess) {
      cudaGetLastError();
      return set_error(AUGSCHED_E_OOM, "step: record buffer allocation failed");
    }
    if (*pp) {
      cudaMemcpyAsync(np, *pp, sizeof(uint32_t) * st.r_n, cudaMemcpyDeviceToDevice, s);
      cudaStreamSynchronize(s);
      cudaFree(*pp);
    }
    *pp = np;
  }
  float* nt = nullptr;
  if (cudaMalloc(&nt, sizeof(float) * cap) != cudaSuccess) {
    cudaGetLastError();
    return set_error(AUGSCHED_E_OOM, "step: record buffer allocation failed");
  }
  if (st.r_ta) {
    cudaMemcpyAsync(nt, st.r_ta, sizeof(float) * st.r_n, cudaMemcpyDeviceToDevice, s);
    cudaStreamSynchronize(s);
    cudaFree(st.r_ta);
  }
  st.r_ta = nt;
  st.r_cap = cap;
  return AUGSCHED_OK;
}

Slots slots_of(StepState& st, const augsched_instance_params* d_ip, uint32_t* d_err) {
  return Slots{st.st, st.V, st.last, st.ctx, st.kv, st.cpu, st.pend, st.A, st.P, st.Aevt, st.Asnap,
               st.coef, d_ip, st.max_active, st.wkv, st.claimA, st.claimB, st.rec_batch, st.gdirty, d_err,
               (st.ti || st.vi || st.minc) ? st.dmark : nullptr, (st.ti || st.vi) ? st.dlist : nullptr, st.dcnt,
               st.ti_ep};
}

}  // namespace

#ifdef AUGSCHED_FM_TIMING
extern "C" AUGSCHED_API int augsched_fm_timing(unsigned long long* host, int reset) {
  if (cudaMemcpyFromSymbol(host, g_fm_t, sizeof(g_fm_t)) != cudaSuccess) return -3;
  if (reset) {
    static const unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_fm_t, z, sizeof(z)) != cudaSuccess) return -3;
  }
  return 0;
}
#endif

static size_t pf_smem_bytes() { return sizeof(unsigned long long) * 2 * PF_SCAP; }
static size_t coop_smem_bytes() {
  // sbuf [PF_SCAP] + the digit counters [CNW][CNB] (16-bit), which the
  // incremental path reuses as the bitonic exchange buffer [PF_SCAP]
  const size_t cnt = sizeof(uint16_t) * CNW * CNB, xch = sizeof(unsigned long long) * PF_SCAP;
  return sizeof(unsigned long long) * PF_SCAP + (cnt > xch ? cnt : xch);
}
static size_t full_multi_smem(int NT, int E) {
  const size_t cnt = sizeof(uint16_t) * 512 * (NT / 32);
  return sizeof(unsigned long long) * 2 * (size_t)NT * E + (cnt > sizeof(SelShm) ? cnt : sizeof(SelShm));
}

int step_ensure(StepState& st, uint32_t n_inst, uint32_t max_active, cudaStream_t s,
                const augsched_config& cfg, const augsched_instance_params* d_ip, uint64_t* launches) {
  if (st.ready) return AUGSCHED_OK;
  const size_t N = (size_t)n_inst * max_active;
  if (N >= (1ull << 30)) return set_error(AUGSCHED_E_CAPACITY, "step: n_instances * max_active must be < 2^30");
  if (max_active >= (1u << 24)) return set_error(AUGSCHED_E_CAPACITY, "step: max_active must be < 2^24");
  st.n_inst = n_inst;
  st.max_active = max_active;
  st.N = N;
  st.n_tiles = (uint32_t)((N + STILE - 1) / STILE);
  // digit passes (LSD): key bits 0-7, 8-15, 16-23, then key bits 24-31 with
  // the tier above them (10 bits), then the instance bytes
  st.npass = 0;
  int hoff = 0;
  auto add = [&](int src, int shift, int bits) {
    st.passes[st.npass++] = PassDesc{src, shift, bits, hoff};
    hoff += 1 << bits;
  };
  add(0, PK_KEY, 8);
  add(0, PK_KEY + 8, 8);
  add(0, PK_KEY + 16, 8);
  add(0, PK_KEY + 24, 10);
  for (uint32_t x = n_inst - 1, b = 0; x > 0; x >>= 8, ++b) add(2, (int)(8 * b), 8);
  if (hoff > STEP_HIST_WORDS) return set_error(AUGSCHED_E_CAPACITY, "step: too many sort passes");
  const size_t zwords = 4 * (size_t)n_inst + STEP_HIST_WORDS + STEP_MAX_PASS + PF_NCNT;
  int rc;
  if ((rc = salloc(st, &st.st, N)) || (rc = salloc(st, &st.V, N)) || (rc = salloc(st, &st.last, N)) ||
      (rc = salloc(st, &st.ctx, N)) || (rc = salloc(st, &st.kv, N)) || (rc = salloc(st, &st.cpu, N)) ||
      (rc = salloc(st, &st.pend, N)) || (rc = salloc(st, &st.A, n_inst)) ||
      (rc = salloc(st, &st.P, n_inst)) || (rc = salloc(st, &st.Aevt, n_inst)) ||
      (rc = salloc(st, &st.Asnap, n_inst)) || (rc = salloc(st, &st.need, n_inst)) ||
      (rc = salloc(st, &st.coef, n_inst)) || (rc = salloc(st, &st.budget, n_inst)) ||
      (rc = salloc(st, &st.zbuf, zwords)) || (rc = salloc(st, &st.admitted, n_inst)) ||
      (rc = salloc(st, &st.flag, n_inst)) || (rc = salloc(st, &st.order, N)) ||
      (rc = salloc(st, &st.grant, N)) || (rc = salloc(st, &st.key, N)) ||
      (rc = salloc(st, &st.k0, N)) || (rc = salloc(st, &st.k1, N)) ||
      (rc = salloc(st, &st.lb_status, (size_t)st.n_tiles << STEP_RB_MAX)) ||
      (rc = salloc(st, &st.lb_gstatus, (size_t)st.n_tiles << STEP_RB_MAX)) ||
      (rc = salloc(st, &st.pf_A, PF_SCAP)) || (rc = salloc(st, &st.pf_C, N)) ||
      (rc = salloc(st, &st.gslot, N)) || (rc = salloc(st, &st.pf_theta, 2 * (size_t)n_inst)) ||
      (rc = salloc(st, &st.pf_H, PF_HCAP)) || (rc = salloc(st, &st.wkv, 1)) ||
      (rc = salloc(st, &st.pf_nact, 2)) || (rc = salloc(st, &st.n_active, n_inst)) ||
      (rc = salloc(st, &st.tier_off, 3 * (size_t)n_inst)) || (rc = salloc(st, &st.claimA, N)) ||
      (rc = salloc(st, &st.claimB, N)) || (rc = salloc(st, &st.gdirty, n_inst)) ||
      (rc = salloc(st, &st.coop_bar, 1)) || (rc = salloc(st, &st.gA, 2)))
    return rc;
  // one memset per full step clears the tier counts, histograms and tile counters
  st.zwords = zwords;
  st.tcnt = st.zbuf;
  st.ghist = st.zbuf + 4 * (size_t)n_inst;
  st.tile_ctr = st.ghist + STEP_HIST_WORDS;
  st.pf_cnt = st.tile_ctr + STEP_MAX_PASS;
  st.pf_epoch = 0;
  st.rec_batch = 0;
  struct Z { void* p; int v; size_t n; };
  const Z zs[] = {
      {st.zbuf, 0, sizeof(uint32_t) * zwords},            // the prefix kernel expects clear counters
      {st.pf_nact, 0, 2 * sizeof(uint32_t)},
      {st.wkv, 0, sizeof(uint32_t)},
      {st.pf_theta, 0xFF, 2 * sizeof(unsigned long long) * (size_t)n_inst},   // no anchor: every slot
      {st.claimA, 0xFF, sizeof(unsigned long long) * N},  // no claim: larger than every key
      {st.claimB, 0xFF, sizeof(unsigned long long) * N},
      {st.gslot, 0, sizeof(uint32_t) * N},
      {st.st, 0, sizeof(uint32_t) * N},
      {st.ctx, 0, sizeof(int32_t) * N},
      {st.kv, 0, sizeof(int32_t) * N},
      {st.cpu, 0, sizeof(int32_t) * N},
      {st.pend, 0, sizeof(int32_t) * N},
      {st.grant, 0, sizeof(uint32_t) * N},                // grant[j] = 0 beyond the admitted prefix
      {st.admitted, 0, sizeof(uint32_t) * n_inst},
      {st.gdirty, 0, sizeof(uint32_t) * n_inst},
      {st.coop_bar, 0, sizeof(unsigned long long)},
      {st.gA, 0, 2 * sizeof(long long)},
      {st.n_active, 0, sizeof(uint32_t) * n_inst},
      {st.tier_off, 0, 3 * sizeof(uint32_t) * n_inst},
      {st.A, 0, sizeof(long long) * n_inst},
      {st.P, 0, sizeof(long long) * n_inst},
      {st.Aevt, 0, sizeof(long long) * n_inst},
      {st.lb_status, 0, sizeof(unsigned long long) * ((size_t)st.n_tiles << STEP_RB_MAX)},
      {st.lb_gstatus, 0, sizeof(unsigned long long) * ((size_t)st.n_tiles << STEP_RB_MAX)},
  };
  for (const Z& z : zs)
    if ((rc = cuda_check(cudaMemsetAsync(z.p, z.v, z.n, s), "step_ensure: clear"))) return rc;
  st.G = 1;
  while ((uint64_t)st.G * st.G < st.n_tiles) ++st.G;   // ~sqrt(tiles) tiles per look-back group
  coef_kernel<<<(n_inst + 255) / 256, 256, 0, s>>>(cfg, d_ip, st.coef, n_inst);
  *launches += 1;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(pf_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pf_smem_bytes());
  {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pf_step_kernel, FNT, pf_smem_bytes());
    st.pf_grid = st.sms * (occ > 0 ? occ : 1);
  }
  cudaFuncSetAttribute(pf_multi_kernel<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PF_MULTI_SMEM);
  if (n_inst == 1) {
    cudaFuncSetAttribute(full_coop_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coop_smem_bytes());
    cudaFuncSetAttribute(full_coop_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coop_smem_bytes());
    int occ = 0, occ_vi = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, full_coop_kernel<false>, CNT, coop_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_vi, full_coop_kernel<true>, CNT, coop_smem_bytes());
    if (occ_vi < 1) st.vi = false;
    // vi checks the order on chunks of <= 8,192 words held in registers (one
    // per CTA but CTA 0): larger queues sort with the plain kernel, whose
    // sort is faster there than a looping merge (measured at 4M / 16M)
    if (N > (size_t)(st.sms - 1) * 8192) st.vi = false;
    st.coop_grid = occ >= 1 ? st.sms : 0;   // one CTA per SM
    st.coop_bar_base = 0;
    if (st.sms < 128 || st.sms > 256) st.coop_grid = 0;   // column scan: <= 4 digits per CTA, one CTA per thread of a 256-thread group
    if (st.coop_grid > 0 && (rc = salloc(st, &st.coop_hist, 4 * ((size_t)st.coop_grid + 1) * CNB))) return rc;
    if ((st.ti || st.vi) && st.coop_grid > 0) {
      if ((rc = salloc(st, &st.tiw, N)) || (rc = salloc(st, &st.tiw2, N)) || (rc = salloc(st, &st.ubuf, N)) ||
          (rc = salloc(st, &st.ti_n, 2)) || (rc = salloc(st, &st.dmark, N)) ||
          (rc = salloc(st, &st.dlist, 2 * (size_t)TI_DCAP)) || (rc = salloc(st, &st.dcnt, 2)) ||
          (rc = salloc(st, &st.ti_misc, 4)) || (rc = salloc(st, &st.ti_gcnt, TI_DCAP + 1)))
        return rc;
      if ((rc = cuda_check(cudaMemsetAsync(st.ti_gcnt, 0, sizeof(uint32_t) * (TI_DCAP + 1), s), "step_ensure: clear")))
        return rc;
      if ((rc = cuda_check(cudaMemsetAsync(st.dmark, 0, sizeof(uint32_t) * N, s), "step_ensure: clear")) ||
          (rc = cuda_check(cudaMemsetAsync(st.dcnt, 0, 2 * sizeof(uint32_t), s), "step_ensure: clear")) ||
          (rc = cuda_check(cudaMemsetAsync(st.ti_n, 0, 2 * sizeof(uint32_t), s), "step_ensure: clear")))
        return rc;
    } else {
      st.ti = false;
      st.vi = false;
    }
  }
  // batched full step: each instance's order is kept for the next step, which
  // merges the changed slots into it (full_multi_kernel)
  st.minc = false;
  st.minc_valid = false;
#ifndef AUGSCHED_NO_MINC
  if (n_inst > 1 && max_active <= 8192) {
    if ((rc = salloc(st, &st.mord, N)) || (rc = salloc(st, &st.mord_n, n_inst)) ||
        (rc = salloc(st, &st.dmark, N)))
      return rc;
    if ((rc = cuda_check(cudaMemsetAsync(st.dmark, 0, sizeof(uint32_t) * N, s), "step_ensure: clear")) ||
        (rc = cuda_check(cudaMemsetAsync(st.mord_n, 0, sizeof(uint32_t) * n_inst, s), "step_ensure: clear")))
      return rc;
    st.minc = true;
  }
#endif
  cudaFuncSetAttribute(pf_multi_kernel<PNT, PF_SCAP / PNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)PF_MULTI_SMEM);
  st.epoch = 0;
  st.ready = true;
  return cuda_check(cudaGetLastError(), "step_ensure");
}

int step_enqueue(StepState& st, uint32_t inst, const augsched_record_soa* r, uint32_t n, int on_dev,
                 cudaStream_t s, uint32_t* d_err, uint64_t* launches) {
  if (n == 0) return AUGSCHED_OK;
  if ((uint64_t)st.r_n + n > 4ull * st.N + 1024)
    return set_error(AUGSCHED_E_CAPACITY, "enqueue: too many pending records");
  const void* srcs[] = {r->kind, r->id, r->la, r->lb, r->lc, r->flags, r->last, r->ctx, r->kv, r->cpu,
                        r->pend, r->ta};
  for (const void* p : srcs)
    if (!p) return set_error(AUGSCHED_E_INVALID, "enqueue: every record column must be non-NULL");
  if (!on_dev) {
    for (uint32_t j = 0; j < n; ++j)
      if (r->kind[j] < AUGSCHED_K_NEW || r->kind[j] > AUGSCHED_K_IMPORT || r->id[j] >= st.max_active)
        return set_error(AUGSCHED_E_INVALID, "enqueue: bad record kind or id");
  }
  int rc = grow_records(st, st.r_n + n, s);
  if (rc) return rc;
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  uint32_t* dst[] = {st.r_kind, st.r_id, st.r_la, st.r_lb, st.r_lc, st.r_flags, st.r_last, st.r_ctx,
                     st.r_kv, st.r_cpu, st.r_pend};
  for (int c = 0; c < 11; ++c) {
    cudaError_t e = cudaMemcpyAsync(dst[c] + st.r_n, srcs[c], sizeof(uint32_t) * n, kind, s);
    if (e != cudaSuccess) return cuda_check(e, "enqueue copy");
  }
  cudaError_t e = cudaMemcpyAsync(st.r_ta + st.r_n, r->ta, sizeof(float) * n, kind, s);
  if (e != cudaSuccess) return cuda_check(e, "enqueue copy");
  rec_fix_kernel<<<(n + 255) / 256, 256, 0, s>>>(st.r_kind + st.r_n, st.r_id + st.r_n, n, inst,
                                                 st.max_active, d_err, st.claimA, st.claimB,
                                                 st.rec_batch + 1, st.r_n);
  *launches += 1;
  st.r_n += n;
  if (!on_dev) {
    // host arrays must be consumed before returning (pageable copies are
    // staged by the driver; a pinned source would not be)
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_check(e, "enqueue sync");
  }
  return cuda_check(cudaGetLastError(), "enqueue");
}

namespace {
// Engine events of the last forward, snapshot, returns / arrivals / imports.
void run_records(StepState& st, Slots S, uint32_t* d_err, uint64_t now, cudaStream_t s,
                 uint64_t* launches) {
  if (!st.r_n) return;
  S.batch = ++st.rec_batch;   // the batch the pending records claimed their slots for
  const uint32_t ni = st.n_inst;
  Rec r{st.r_kind, st.r_id, st.r_la, st.r_lb, st.r_lc, st.r_flags, st.r_last, st.r_ctx, st.r_kv,
        st.r_cpu, st.r_pend, st.r_ta};
  const uint32_t g = (st.r_n + 255) / 256;
  rec_phaseA<<<g, 256, 0, s>>>(r, st.r_n, S, d_err);
  snap_kernel<<<(ni + 255) / 256, 256, 0, s>>>(st.A, st.Asnap, ni);
  rec_phaseBC<<<g, 256, 0, s>>>(r, st.r_n, S, now, d_err);
  *launches += 3;
  st.r_n = 0;
}

}  // namespace


// Time-invariant handles: the step epoch of the dirty marks, and the clear
// of the consumed list after the step's kernels.
static void ti_begin(StepState& st) {
  if (st.ti || st.vi || st.minc) ++st.ti_ep;
}
static int ti_end(StepState& st, cudaStream_t s) {
  if (!st.ti && !st.vi) return AUGSCHED_OK;
  return cuda_check(cudaMemsetAsync(st.dcnt + (st.ti_ep & 1), 0, sizeof(uint32_t), s), "step: clear");
}

int step_run_prefix(StepState& st, const augsched_config& cfg, int64_t cap,
                    const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
                    augsched_step_out* out, cudaStream_t s, uint64_t* launches) {
  st.minc_valid = false;   // the batched full step's kept order does not see this step's changes
  // the prefix selection is bounded by PF_SCAP; several instances need their
  // slots on chip (one CTA per instance)
  uint32_t scap = 32;
  while (scap < st.max_limit) scap <<= 1;
  const size_t msmem = sizeof(unsigned long long) * ((size_t)st.max_active + 2 * (size_t)scap);
  if (st.max_limit > PF_SCAP || (st.n_inst > 1 && msmem > PF_MULTI_SMEM))
    return step_run(st, cfg, cap, d_ip, d_err, now, out, s, launches);
  ti_begin(st);
  Slots S = slots_of(st, d_ip, d_err);
  // a prefix step leaves no full order, so the next full step sorts: no
  // change of this step needs a dirty mark
  S.dmark = nullptr;
  S.dlist = nullptr;
  run_records(st, S, d_err, now, s, launches);
  st.ti_valid = false;   // no full order: the next full step sorts
  if (st.n_inst > 1) {
#ifndef AUGSCHED_PF_MULTI_SMALL
#define AUGSCHED_PF_MULTI_SMALL (4 * 256)
#endif
    if (scap <= AUGSCHED_PF_MULTI_SMALL)   // small limits: 256-thread CTAs, more instances resident per SM
      pf_multi_kernel<256, 4><<<st.n_inst, 256, msmem, s>>>(S, cfg, cap, now, st.budget, st.n_active, st.order,
                                                             st.key, st.grant, st.admitted, st.gslot, scap, st.pf_theta);
    else
      pf_multi_kernel<PNT, PF_SCAP / PNT><<<st.n_inst, PNT, msmem, s>>>(S, cfg, cap, now, st.budget, st.n_active,
                                                                        st.order, st.key, st.grant, st.admitted,
                                                                        st.gslot, scap, st.pf_theta);
    *launches += 1;
    out->budget = reinterpret_cast<const int64_t*>(st.budget);
    out->n_active = st.n_active;
    out->admitted = st.admitted;
    out->order = st.order;
    out->grant = st.grant;
    out->key = st.key;
    out->tier_off = nullptr;
    return cuda_check(cudaGetLastError(), "step_prefix");
  }
  // no memset: the kernel leaves its counters cleared for the next call
  // (a full step in between leaves its histograms behind: clear once)
  if (st.pf_dirty) {
    const int rc = cuda_check(cudaMemsetAsync(st.zbuf, 0, sizeof(uint32_t) * st.zwords, s), "step_prefix: clear");
    if (rc) return rc;
    st.pf_dirty = false;
  }
  if (++st.pf_epoch >= (1u << 30)) st.pf_epoch = 1;
  const uint32_t ep = st.pf_epoch;
  PfArgs pa{};
  pa.S = S; pa.cfg = cfg; pa.cap = cap; pa.now = now; pa.N = (uint32_t)st.N; pa.spec = st.pf_spec ? 1 : 0;
  pa.k0 = st.k0; pa.A = st.pf_A; pa.C = st.pf_C; pa.theta = st.pf_theta; pa.H = st.pf_H; pa.ghist = st.ghist;
  pa.cnt = st.pf_cnt; pa.ep = ep; pa.n_active = st.pf_nact + (ep & 1u); pa.n_active_next = st.pf_nact + ((ep + 1u) & 1u);
  pa.budget = st.budget;
  pa.order = st.order; pa.keyout = st.key; pa.grant = st.grant; pa.admitted = st.admitted; pa.gslot = st.gslot;
  void* args[] = {&pa};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&pf_step_kernel), st.pf_grid, FNT,
                                              args, pf_smem_bytes(), s);
  if (e != cudaSuccess) return cuda_check(e, "step_prefix: cooperative launch");
  *launches += 1;
  {
    const int rc2 = ti_end(st, s);
    if (rc2) return rc2;
  }
  out->budget = reinterpret_cast<const int64_t*>(st.budget);
  out->n_active = pa.n_active;
  out->admitted = st.admitted;
  out->order = st.order;
  out->grant = st.grant;
  out->key = st.key;
  out->tier_off = nullptr;
  return cuda_check(cudaGetLastError(), "step_prefix");
}

template <int NT, int E>
static void launch_full_multi(const StepState& st, const Slots& S, const augsched_config& cfg, int64_t cap,
                              uint64_t now, cudaStream_t s) {
  const size_t smem = full_multi_smem(NT, E);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(full_multi_kernel<NT, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  full_multi_kernel<NT, E><<<st.n_inst, NT, smem, s>>>(S, cfg, cap, now, st.budget, st.n_active, st.tier_off,
                                                        st.order, st.key, st.grant, st.admitted, st.gslot,
                                                        st.mord, st.mord_n, st.minc_valid ? 1 : 0);
}

int step_run(StepState& st, const augsched_config& cfg, int64_t cap,
             const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
             augsched_step_out* out, cudaStream_t s, uint64_t* launches) {
  ti_begin(st);
  Slots S = slots_of(st, d_ip, d_err);
  const uint32_t ni = st.n_inst;
  run_records(st, S, d_err, now, s, launches);
#ifndef AUGSCHED_NO_FULL_COOP
  // one instance: one cooperative kernel (keys, four sort passes with grid
  // barriers, admission by CTA 0)
  if (ni == 1 && st.max_limit <= PF_SCAP && st.coop_grid > 0) {
    CoopArgs ca{};
    ca.S = S; ca.cfg = cfg; ca.cap = cap; ca.now = now; ca.N = (uint32_t)st.N; ca.max_limit = st.max_limit;
    ca.kA = st.k0; ca.kB = st.k1; ca.kpre = st.pf_A; ca.hist = st.coop_hist; ca.bar = st.coop_bar;
    ca.tot = st.coop_hist + 4 * (size_t)st.coop_grid * CNB;
    ca.bar_base = st.coop_bar_base;
    ca.budget = st.budget; ca.n_active = st.n_active; ca.tier_off = st.tier_off; ca.order = st.order;
    ca.keyout = st.key; ca.grant = st.grant; ca.admitted = st.admitted; ca.gslot = st.gslot;
    const uint32_t cur = st.ti_ep & 1;
    ca.ti = st.ti ? 1 : 0;
    ca.vi = st.vi ? 1 : 0;
    ca.ti_try = (st.ti || st.vi) && st.ti_valid ? 1 : 0;
    ca.tiw_in = st.tiw; ca.tiw_out = st.tiw2; ca.ubuf = st.ubuf;
    ca.ti_n_in = st.ti_n ? st.ti_n + (cur ^ 1) : nullptr;
    ca.ti_n_out = st.ti_n ? st.ti_n + cur : nullptr;
    ca.ti_misc = st.ti_misc;
    ca.gcnt = st.ti_gcnt;
    void* args[] = {&ca};
    const void* kfn = st.vi ? reinterpret_cast<const void*>(&full_coop_kernel<true>)
                            : reinterpret_cast<const void*>(&full_coop_kernel<false>);
    cudaError_t e = cudaLaunchCooperativeKernel(kfn, st.coop_grid,
                                                CNT, args, coop_smem_bytes(), s);
    if (e != cudaSuccess) return cuda_check(e, "step: cooperative launch");
    if (st.ti || st.vi) {   // the sorted words of this order are the next step's input
      std::swap(st.tiw, st.tiw2);
      st.ti_valid = true;
      int rc2 = ti_end(st, s);
      if (rc2) return rc2;
    }
    st.coop_bar_base += 12ull * (unsigned long long)st.coop_grid;   // twelve grid barriers per call
    *launches += 1;
    out->budget = reinterpret_cast<const int64_t*>(st.budget);
    out->n_active = st.n_active;
    out->admitted = st.admitted;
    out->order = st.order;
    out->grant = st.grant;
    out->key = st.key;
    out->tier_off = st.tier_off;
    return cuda_check(cudaGetLastError(), "step (cooperative)");
  }
#endif
#ifndef AUGSCHED_NO_FULL_MULTI
  // several instances whose slots fit in one CTA's shared memory: one CTA
  // per instance sorts and admits (no device-wide pass)
  if (ni > 1 && st.max_active <= 8192) {
    const uint32_t MA = st.max_active;
    if (MA <= 256) launch_full_multi<256, 1>(st, S, cfg, cap, now, s);
    else if (MA <= 512) launch_full_multi<256, 2>(st, S, cfg, cap, now, s);
    else if (MA <= 1024) launch_full_multi<256, 4>(st, S, cfg, cap, now, s);
    else if (MA <= 2048) launch_full_multi<256, 8>(st, S, cfg, cap, now, s);
    else if (MA <= 4096) launch_full_multi<256, 16>(st, S, cfg, cap, now, s);
    else launch_full_multi<512, 16>(st, S, cfg, cap, now, s);
    st.minc_valid = st.minc;   // this step's order is the next one's starting point
    *launches += 1;
    out->budget = reinterpret_cast<const int64_t*>(st.budget);
    out->n_active = st.n_active;
    out->admitted = st.admitted;
    out->order = st.order;
    out->grant = st.grant;
    out->key = st.key;
    out->tier_off = st.tier_off;
    return cuda_check(cudaGetLastError(), "step (batched)");
  }
#endif
  st.pf_dirty = true;
  int rc = cuda_check(cudaMemsetAsync(st.zbuf, 0, sizeof(uint32_t) * st.zwords, s), "step: clear");
  if (rc) return rc;
  KeyArgs ka{};
  ka.S = S; ka.cfg = cfg; ka.cap = cap; ka.now = now; ka.k0 = st.k0;
  ka.ghist = st.ghist; ka.tcnt = st.tcnt; ka.budget = st.budget; ka.npass = st.npass;
  for (int p = 0; p < st.npass; ++p) ka.passes[p] = st.passes[p];
  ka.N = (uint32_t)st.N;
  const size_t kblocks = (st.N + KNT * KU - 1) / (KNT * KU);
  const int kgrid = (int)(kblocks < (size_t)st.sms * 8 ? kblocks : (size_t)st.sms * 8);
  keys_kernel<<<kgrid, KNT, 0, s>>>(ka);
  *launches += 1;
  unsigned long long *kin = st.k0, *kout = st.k1;
  for (int p = 0; p < st.npass; ++p) {
    SortArgs sa{};
    sa.kin = kin; sa.kout = kout; sa.n = (uint32_t)st.N; sa.d = st.passes[p];
    sa.MA = st.max_active; sa.ghist = st.ghist + st.passes[p].hoff; sa.status = st.lb_status;
    sa.gstatus = st.lb_gstatus; sa.G = st.G;
    sa.epoch = ++st.epoch & ((1ull << 30) - 1); sa.tile_ctr = st.tile_ctr + p;
    sa.final_ = p == st.npass - 1;
    sa.order = st.order; sa.keyout = st.key;
    if (st.passes[p].bits == 10) sort_pass_kernel<10><<<st.n_tiles, SNT, 0, s>>>(sa);
    else sort_pass_kernel<8><<<st.n_tiles, SNT, 0, s>>>(sa);
    *launches += 1;
    unsigned long long* t = kin; kin = kout; kout = t;
  }
  admit_kernel<<<ni, ANT, 0, s>>>(S, cfg, cap, now, st.budget, st.tcnt, st.n_active, st.tier_off, st.order,
                                  st.grant, st.admitted);
  *launches += 1;
  st.ti_valid = false;
  {
    const int rc2 = ti_end(st, s);
    if (rc2) return rc2;
  }
  out->budget = reinterpret_cast<const int64_t*>(st.budget);
  out->n_active = st.n_active;
  out->admitted = st.admitted;
  out->order = st.order;
  out->grant = st.grant;
  out->key = st.key;
  out->tier_off = st.tier_off;
  return cuda_check(cudaGetLastError(), "step");
}

// ---- sharded single queue (f4) ----------------------------------------------
static uint32_t shard_ocap(const StepState& st) {
  uint32_t c = 32;
  while (c < st.max_limit) c <<= 1;
  return c;
}
size_t step_shard_offer_bytes(const StepState& st) { return shard_offer_bytes(shard_ocap(st)); }

int step_shard_begin(StepState& st, const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
                     int64_t* ledger, cudaStream_t s, uint64_t* launches) {
  if (st.n_inst != 1 || st.coop_grid <= 0 || st.max_limit > PF_SCAP)
    return set_error(AUGSCHED_E_INVALID, "shard: needs a single-instance handle with limits <= 8192 on a GPU "
                                         "that runs the cooperative step");
  ti_begin(st);
  Slots S = slots_of(st, d_ip, d_err);
  // CALL / FINISH of the last forward: C_other of the issued calls from the
  // GLOBAL ledger before the events (R13; every shard holds it after the
  // last commit); the caller all-reduces this shard's A after them into the
  // global snapshot A_snap (S1) that the intake of shard_offer uses
  S.Aevt = st.gA;
  st.shard_batch = st.r_n ? ++st.rec_batch : 0u;
  if (st.r_n) {
    S.batch = st.shard_batch;
    Rec r{st.r_kind, st.r_id, st.r_la, st.r_lb, st.r_lc, st.r_flags, st.r_last, st.r_ctx, st.r_kv,
          st.r_cpu, st.r_pend, st.r_ta};
    rec_phaseA<<<(st.r_n + 255) / 256, 256, 0, s>>>(r, st.r_n, S, d_err);
    *launches += 1;
  }
  st.shard_now = now;
  int rc;
  if ((rc = cuda_check(cudaMemcpyAsync(ledger, st.A, sizeof(long long), cudaMemcpyDeviceToDevice, s), "shard")) ||
      (rc = cuda_check(cudaMemcpyAsync(ledger + 1, st.P, sizeof(long long), cudaMemcpyDeviceToDevice, s), "shard")))
    return rc;
  return cuda_check(cudaGetLastError(), "shard_begin");
}

int step_shard_offer(StepState& st, const augsched_config& cfg, int64_t cap, const augsched_instance_params* d_ip,
                     uint32_t* d_err, const int64_t* ledger_sum, void* offer, cudaStream_t s, uint64_t* launches) {
  Slots S = slots_of(st, d_ip, d_err);
  if (st.r_n) {   // RETURN / NEW / IMPORT against the global snapshot A_snap = ledger_sum[0]
    S.batch = st.shard_batch;
    S.Asnap = const_cast<long long*>(reinterpret_cast<const long long*>(ledger_sum));
    Rec r{st.r_kind, st.r_id, st.r_la, st.r_lb, st.r_lc, st.r_flags, st.r_last, st.r_ctx, st.r_kv,
          st.r_cpu, st.r_pend, st.r_ta};
    rec_phaseBC<<<(st.r_n + 255) / 256, 256, 0, s>>>(r, st.r_n, S, st.shard_now, d_err);
    *launches += 1;
    st.r_n = 0;
    S = slots_of(st, d_ip, d_err);
  }
  const uint32_t ocap = shard_ocap(st);
  int rc = cuda_check(cudaMemsetAsync(offer, 0, sizeof(ShardHdr), s), "shard_offer: clear");
  if (rc) return rc;
  CoopArgs ca{};
  ca.S = S; ca.cfg = cfg; ca.cap = cap; ca.now = st.shard_now; ca.N = (uint32_t)st.N; ca.max_limit = st.max_limit;
  ca.kA = st.k0; ca.kB = st.k1; ca.kpre = st.pf_A; ca.hist = st.coop_hist; ca.bar = st.coop_bar;
  ca.tot = st.coop_hist + 4 * (size_t)st.coop_grid * CNB;
  ca.bar_base = st.coop_bar_base;
  ca.budget = st.budget; ca.n_active = st.n_active; ca.tier_off = st.tier_off; ca.order = st.order;
  ca.keyout = st.key; ca.grant = st.grant; ca.admitted = st.admitted; ca.gslot = st.gslot;
  const uint32_t cur = st.ti_ep & 1;
  ca.ti = st.ti ? 1 : 0;
  ca.vi = st.vi ? 1 : 0;
  ca.ti_try = (st.ti || st.vi) && st.ti_valid ? 1 : 0;
  ca.tiw_in = st.tiw; ca.tiw_out = st.tiw2; ca.ubuf = st.ubuf;
  ca.ti_n_in = st.ti_n ? st.ti_n + (cur ^ 1) : nullptr;
  ca.ti_n_out = st.ti_n ? st.ti_n + cur : nullptr;
  ca.ti_misc = st.ti_misc;
  ca.gcnt = st.ti_gcnt;
  ca.ledger = nullptr;            // the limit is the commit's (global ledger); the offer holds min(n, ocap)
  st.shard_ledger = ledger_sum;
  ca.offer = static_cast<unsigned char*>(offer);
  ca.ocap = ocap;
  void* args[] = {&ca};
  const void* kfn = st.vi ? reinterpret_cast<const void*>(&full_coop_kernel<true>)
                          : reinterpret_cast<const void*>(&full_coop_kernel<false>);
  cudaError_t e = cudaLaunchCooperativeKernel(kfn, st.coop_grid,
                                              CNT, args, coop_smem_bytes(), s);
  if (e != cudaSuccess) return cuda_check(e, "shard_offer: cooperative launch");
  st.coop_bar_base += 12ull * (unsigned long long)st.coop_grid;
  shard_holders_kernel<<<(uint32_t)((st.N + 255) / 256), 256, 0, s>>>(S, st.shard_now, (uint32_t)st.N,
                                                                       static_cast<unsigned char*>(offer), ocap);
  *launches += 2;
  if (st.ti || st.vi) {
    std::swap(st.tiw, st.tiw2);
    st.ti_valid = true;
    if ((rc = ti_end(st, s))) return rc;
  }
  return cuda_check(cudaGetLastError(), "shard_offer");
}

int step_shard_commit(StepState& st, const augsched_config& cfg, int64_t cap, const augsched_instance_params* d_ip,
                      uint32_t* d_err, const int64_t* ledger_sum, const void* offers, uint32_t n_ranks,
                      uint32_t rank, augsched_step_out* out, cudaStream_t s, uint64_t* launches) {
  if (n_ranks == 0 || rank >= n_ranks || (uint64_t)n_ranks * st.max_active >= (1ull << 30))
    return set_error(AUGSCHED_E_INVALID, "shard_commit: bad rank count / rank, or ranks x max_active >= 2^30");
  Slots S = slots_of(st, d_ip, d_err);
  CommitArgs ca{};
  ca.S = S; ca.cfg = cfg; ca.cap = cap; ca.now = st.shard_now;
  ca.offers = static_cast<const unsigned char*>(offers);
  ca.ocap = shard_ocap(st);
  ca.obytes = shard_offer_bytes(ca.ocap);
  ca.n_ranks = n_ranks; ca.rank = rank; ca.MA = st.max_active;
  (void)ledger_sum;
  ca.gledger = st.gA;
  ca.budget = st.budget; ca.n_active = st.n_active; ca.admitted = st.admitted; ca.order = st.order;
  ca.keyout = st.key; ca.grant = st.grant; ca.err = d_err;
  static bool attr = false;
  const size_t smem = 2 * sizeof(unsigned long long) * PF_SCAP;
  if (!attr) {
    cudaFuncSetAttribute(shard_commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  shard_commit_kernel<<<1, 1024, smem, s>>>(ca);
  *launches += 1;
  out->budget = reinterpret_cast<const int64_t*>(st.budget);
  out->n_active = st.n_active;
  out->admitted = st.admitted;
  out->order = st.order;
  out->grant = st.grant;
  out->key = st.key;
  out->tier_off = nullptr;
  return cuda_check(cudaGetLastError(), "shard_commit");
}

void step_free(StepState& st) {
  for (int i = 0; i < st.n_alloc; ++i) cudaFree(st.alloc_list[i]);
  st.n_alloc = 0;
  uint32_t* u[] = {st.r_kind, st.r_id, st.r_la, st.r_lb, st.r_lc, st.r_flags, st.r_last, st.r_ctx,
                   st.r_kv, st.r_cpu, st.r_pend};
  for (auto p : u)
    if (p) cudaFree(p);
  if (st.r_ta) cudaFree(st.r_ta);
  st = StepState();
}

}  // namespace augsched
