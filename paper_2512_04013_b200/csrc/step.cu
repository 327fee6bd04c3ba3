// augsched_step kernels (see step.cuh).  sm_100a, compiled with -fmad=false.
#include <cuda_runtime.h>
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

// convert per-instance ids to global slot indices and validate kinds/ids
__global__ void rec_fix_kernel(const uint32_t* kind, uint32_t* id, uint32_t n, uint32_t inst,
                               uint32_t MA, uint32_t* err) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t k = kind[j], x = id[j];
  if (k < AUGSCHED_K_NEW || k > AUGSCHED_K_IMPORT || x >= MA) {
    flag_err(err, 1u);
    id[j] = 0xffffffffu;
    return;
  }
  id[j] = inst * MA + x;
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
};

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
  const uint32_t inst = g / S.MA;
  const uint32_t st = S.st[g] & 15;
  if (k == AUGSCHED_K_FINISH) {
    if (st < ST_RUN || st > ST_WAIT) { flag_err(err, 1u); return; }
    ledger_add(&S.A[inst], -(long long)S.kv[g]);
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
  // IMPORT
  const uint32_t f = r.flags[j];
  const uint32_t ns = (f >> 4) & 7, pol = (f >> 8) & 3;
  const bool st2 = (f >> 12) & 1;
  if (ns < ST_RUN || ns > ST_PAUSED || pol > 2) { flag_err(err, 1u); return; }
  S.V[g] = st2 ? intake_stage2(c, pm, (int)pol, r.la[j], r.lb[j], r.lc[j], (double)r.ta[j], flag1, Asnap)
               : intake_stage1(c, pm, r.la[j], r.lb[j], (double)r.ta[j], flag1, Asnap);
  S.st[g] = ns | (pol << 4);
  S.last[g] = r.last[j];
  S.ctx[g] = (int32_t)r.ctx[j]; S.kv[g] = (int32_t)r.kv[j]; S.cpu[g] = (int32_t)r.cpu[j];
  S.pend[g] = (int32_t)r.pend[j];
  if (ns == ST_PAUSED && pol == POL_P) ledger_add(&S.P[inst], (long long)r.kv[j]);
  else ledger_add(&S.A[inst], (long long)r.kv[j]);
}

// ------------------------------------------------------------------ keys
struct KeyArgs {
  Slots S;
  augsched_config cfg;
  int64_t cap;
  uint64_t now;
  unsigned long long* k0;
  uint32_t* ghist;
  uint32_t* n_active;
  long long* budget;
  int npass;
  PassDesc passes[STEP_MAX_PASS];
  uint32_t N;
  uint32_t* pf_cnt;   // prefix step: [|A|, |C|, b*, below, blocks done]; nullptr otherwise
};

// Packed sort word of one slot: tier:2 | key:32 | slot:30 (tier 3 = not queued).
constexpr int PK_KEY = 30;
constexpr int PK_TIER = 62;
constexpr uint32_t SLOT_MASK = (1u << 30) - 1;

__device__ __forceinline__ uint32_t digit_of(unsigned long long x, const PassDesc& d, uint32_t MA) {
  if (d.src == 0) return (uint32_t)(x >> d.shift) & ((1u << d.bits) - 1u);
  return ((((uint32_t)x & SLOT_MASK) / MA) >> d.shift) & 255u;
}

// Score every slot (a4): key = orderable u32 of fp32(V - alpha*wait) for
// queued slots (tier 0 running, 1 swapped, 2 waiting); empty / paused slots
// get tier 3 and sort behind their instance's queue.  Also the token limit of
// each instance (a3), its queue size and the digit histograms of every sort
// pass (warp-aggregated shared atomics).
constexpr int KCNT = 1024;   // per-block instance-count table of the keys kernel

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
  __shared__ uint32_t wsum[KNT / 32];
  __shared__ uint32_t ticket;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  const bool local_cnt = c1 > c0 && (c1 - 1) / MA - i0 < (uint32_t)KCNT;
  uint32_t myq = 0;   // queued slots seen by this thread (single-instance handles)
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
          myq += tier < 3;
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
      // queued count per instance
      const bool q = valid && tier < 3;
      {
        const unsigned qm = __ballot_sync(FULL, q);
        if (qm) {
          const unsigned peers = __match_any_sync(FULL, q ? (int)inst : -1) & qm;
          if (q && lane == __ffs(peers) - 1) {
            if (local_cnt) atomicAdd(&qcnt[inst - i0], (unsigned)__popc(peers));
            else atomicAdd(&a.n_active[inst], (unsigned)__popc(peers));
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
    for (int o = 16; o > 0; o >>= 1) myq += __shfl_xor_sync(FULL, myq, o);
    if (lane == 0) atomicAdd(&qcnt[0], myq);
  }
  __syncthreads();
  for (int b = tid; b < hw; b += KNT)
    if (h[b]) atomicAdd(&a.ghist[b], h[b]);
  if (local_cnt)
    for (uint32_t b = tid; b <= (c1 - 1) / MA - i0; b += KNT)
      if (qcnt[b]) atomicAdd(&a.n_active[i0 + b], qcnt[b]);
  if (!a.pf_cnt) return;
  // prefix step: the last block locates the bucket b* of the top digit that
  // holds the target-th smallest entry (target = min(B, queued))
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(&a.pf_cnt[4], 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  constexpr int NB = 1 << PF_BITS, PER = NB / KNT;
  const long long B = ld_ll(a.budget);
  const uint32_t nq = __ldcg(&a.n_active[0]);
  const uint32_t target = B <= 0 ? 0u : ((unsigned long long)B < nq ? (uint32_t)B : nq);
  uint32_t loc[PER], sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) { loc[j] = __ldcg(&a.ghist[tid * PER + j]); sum += loc[j]; }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  if (tid == 0) { a.pf_cnt[2] = NB; a.pf_cnt[3] = 0; }
  __syncthreads();
  uint32_t run = inc - sum;
  for (int w = 0; w < warp; ++w) run += wsum[w];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (target > 0 && run < target && run + loc[j] >= target) { a.pf_cnt[2] = tid * PER + j; a.pf_cnt[3] = run; }
    run += loc[j];
  }
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
  unsigned long long base = 0, tot = 0;
  for (int w = 0; w < NW; ++w) {
    const unsigned long long v = wsum[w];
    if (w < warp) base += v;
    tot += v;
  }
  *total = tot;
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
__global__ void __launch_bounds__(ANT) admit_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                    const long long* budget, const uint32_t* n_active,
                                                    const uint32_t* order, uint32_t* grant,
                                                    uint32_t* admitted) {
  __shared__ unsigned long long wsum[ANW];
  __shared__ SelShm sel;
  __shared__ unsigned long long freed;
  const uint32_t i = blockIdx.x;
  const int tid = threadIdx.x;
  const uint32_t MA = S.MA;
  const size_t base = (size_t)i * MA;
  const long long B = budget[i];
  const uint32_t n = n_active[i];
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
  unsigned long long tot;
  block_incl_scan_u64<ANT>(dA, wsum, &tot);
  if (tid == 0) {
    admitted[i] = adm;
    const long long a = ld_ll(&S.A[i]) + (long long)tot;
    S.A[i] = a;
    S.Aevt[i] = a;
  }
}


// ====================================================================== prefix step
// augsched_step_prefix: the same decision round, producing the order only
// for the admitted prefix.  Every queued request has demand >= 1, so the
// admitted prefix lies within the first min(B, n) entries of the order; it
// is found by a count-based selection instead of a full sort:
//   keys_kernel   packed words + histogram of the top 12-bit digit
//   pf_collect    every block locates the bucket b* holding the target-th
//                 entry; words below b* -> A (< target of them), in b* -> C
//   pf_admit      one block: the (target - |A|) smallest of C by a weighted
//                 radix select (weights 1), bitonic sort of the prefix in
//                 shared memory, admission (R17), resolution (R20, exact:
//                 selections over all slots), grant accounting.

__device__ __forceinline__ uint32_t pf_target(long long B, uint32_t n) {
  if (B <= 0) return 0u;
  return (unsigned long long)B < n ? (uint32_t)B : n;
}

__global__ void __launch_bounds__(KNT) pf_collect_kernel(const unsigned long long* k0, uint32_t N,
                                                         uint32_t* cnt, unsigned long long* A,
                                                         unsigned long long* C) {
  const int tid = threadIdx.x, lane = tid & 31;
  constexpr int NB = 1 << PF_BITS;
  const uint32_t bstar = cnt[2];   // written by the last keys_kernel block
  if (bstar >= NB) return;         // nothing to admit
  const unsigned lt = (1u << lane) - 1;
  for (uint32_t base = blockIdx.x * KNT * KU; base < N; base += gridDim.x * KNT * KU) {
    unsigned long long x[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint32_t s = base + u * KNT + tid;
      x[u] = s < N ? k0[s] : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint32_t d = (uint32_t)(x[u] >> (64 - PF_BITS));
      const bool queued = (x[u] >> PK_TIER) < 3;
      const bool inA = queued && d < bstar, inC = queued && d == bstar;
      const unsigned ma = __ballot_sync(FULL, inA), mc = __ballot_sync(FULL, inC);
      if (!(ma | mc)) continue;
      uint32_t ba = 0, bc = 0;
      if (lane == 0) {
        if (ma) ba = atomicAdd(&cnt[0], (unsigned)__popc(ma));
        if (mc) bc = atomicAdd(&cnt[1], (unsigned)__popc(mc));
      }
      ba = __shfl_sync(FULL, ba, 0);
      bc = __shfl_sync(FULL, bc, 0);
      if (inA) A[ba + __popc(ma & lt)] = x[u];
      if (inC) C[bc + __popc(mc & lt)] = x[u];
    }
  }
}

constexpr int PNT = 1024;

// The admitted prefix of instance `inst` from `mt` candidate words in sbuf
// (which hold its first `target` order entries): bitonic sort, admission
// (R17), resolution by exact selections over the instance's slots (R20),
// grant accounting.  `keys` are the instance's packed words (local slot in
// the low bits; tier 3 = not queued); `xch` is a second buffer of the same
// size as sbuf for the sort's shared-memory exchanges.
template <int NT, int EM>
__device__ void pf_finish(const Slots& S, const augsched_config& cfg, int64_t cap, uint64_t now, uint32_t inst,
                          size_t base, const unsigned long long* keys, unsigned long long* sbuf,
                          unsigned long long* xch, uint32_t mt, uint32_t target, long long B, uint32_t* order,
                          uint32_t* keyout, uint32_t* grant, uint32_t* admitted, uint32_t* gslot, SelShm& sel,
                          unsigned long long* wsum, unsigned long long& freed) {
  const int tid = threadIdx.x;
  const uint32_t MA = S.MA;
  // ---- bitonic sort of the prefix (padded to a power of two).  Each thread
  // holds E = P2 / NT elements (index tid + e * NT) in registers: partner
  // distances j < 32 exchange by warp shuffles, j >= NT inside the thread,
  // and only 32 <= j < NT goes through shared memory (double-buffered, one
  // barrier per stage).
  uint32_t P2 = 1;
  while (P2 < mt) P2 <<= 1;
  if (P2 < 32) P2 = 32;
  constexpr int EMAX = EM;
  const uint32_t E = P2 > NT ? P2 / NT : 1u;
  unsigned long long v[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    const uint32_t idx = tid + e * NT;
    v[e] = (e < (int)E && idx < mt) ? sbuf[idx] : ~0ull;
  }
  __syncthreads();
  int xp = 0;
  for (uint32_t k = 2; k <= P2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j < 32) {
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          if (e >= (int)E) break;
          const unsigned long long pv = __shfl_xor_sync(FULL, v[e], j);
          const uint32_t idx = tid + e * NT;
          const bool keep_min = ((idx & j) == 0) == ((idx & k) == 0);
          v[e] = keep_min ? (pv < v[e] ? pv : v[e]) : (pv > v[e] ? pv : v[e]);
        }
      } else if (j < NT) {
        unsigned long long* xbuf = xp ? xch : sbuf;
        xp ^= 1;
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
          if (e < (int)E && tid + e * NT < P2) xbuf[tid + e * NT] = v[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          if (e >= (int)E) break;
          const uint32_t idx = tid + e * NT;
          if (idx >= P2) continue;
          const unsigned long long pv = xbuf[idx ^ j];
          const bool keep_min = ((idx & j) == 0) == ((idx & k) == 0);
          v[e] = keep_min ? (pv < v[e] ? pv : v[e]) : (pv > v[e] ? pv : v[e]);
        }
      } else {
        // partner inside the thread: e ^ (j / NT), unrolled so v stays in registers
#pragma unroll
        for (int bsh = 0; (1 << bsh) < EMAX; ++bsh) {
          if (j != ((uint32_t)NT << bsh)) continue;
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            const int e2 = e ^ (1 << bsh);
            if (e2 <= e || e2 >= (int)E) continue;
            const uint32_t idx = tid + e * NT;
            const bool up = (idx & k) == 0;
            const unsigned long long x0 = v[e], x1 = v[e2];
            if ((x0 > x1) == up) { v[e] = x1; v[e2] = x0; }
          }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    const uint32_t idx = tid + e * NT;
    if (e < (int)E && idx < P2) sbuf[idx] = v[e];
  }
  __syncthreads();
  const uint32_t m = target;
  // ---- a6 admission over the prefix (P_{j-1} < B, partial last, R17)
  unsigned long long Prun = 0, gsum = 0;
  uint32_t adm = 0;
  for (uint32_t j0 = 0; j0 < m && (long long)Prun < B; j0 += NT) {
    const uint32_t j = j0 + tid;
    unsigned long long d = 0;
    uint32_t slot = 0;
    if (j < m) {
      slot = (uint32_t)sbuf[j] & SLOT_MASK;
      d = slot_demand(S, (uint32_t)(base + slot), cfg.s_in);
    }
    unsigned long long tot;
    const unsigned long long inc = block_incl_scan_u64<NT>(d, wsum, &tot);
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
  long long fr = cap - ld_ll(&S.A[inst]) - ld_ll(&S.P[inst]);
  // ---- a7 resolution (rare; exact selections over every slot)
  if ((long long)need > fr) {
    if (tid == 0) freed = 0;
    auto getp = [&](uint32_t x, uint64_t& key, uint32_t& w) {
      const uint32_t stv = S.st[base + x];
      const int32_t kv = S.kv[base + x];
      if ((stv & 15) != ST_PAUSED || ((stv >> 4) & 3) != POL_P || kv <= 0) return false;
      key = ((uint64_t)(0xFFFFFFFFu - (uint32_t)kv) << 24) | x;
      w = (uint32_t)kv;
      return true;
    };
    wselect<NT>(sel, MA, (uint64_t)((long long)need - fr), 56, getp);
    {
      const bool f0 = sel.r.found != 0;
      const uint64_t kd = sel.r.k;
      for (uint32_t x = tid; x < MA; x += NT) {
        uint64_t key;
        uint32_t w;
        if (getp(x, key, w) && (!f0 || key <= kd)) {
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
      auto gete = [&](uint32_t x, uint64_t& key, uint32_t& w) {
        const unsigned long long kx = keys[x];
        if ((kx >> PK_TIER) >= 3) return false;
        const uint32_t g = gslot[base + x];
        w = (uint32_t)S.kv[base + x] + (g == 0xFFFFFFFFu ? 0u : g);
        key = ~kx;
        return w > 0;
      };
      wselect<NT>(sel, MA, (uint64_t)((long long)need - fr), 64, gete);
      const bool f1 = sel.r.found != 0;
      const uint64_t k1 = sel.r.k;
      __syncthreads();
      long long dA = 0;
      for (uint32_t x = tid; x < MA; x += NT) {
        uint64_t key;
        uint32_t w;
        if (gete(x, key, w) && (!f1 || key <= k1)) {
          dA -= S.kv[base + x];
          S.kv[base + x] = 0;
          S.cpu[base + x] = 0;
          S.st[base + x] = ST_WAIT | (S.st[base + x] & 0x30u);
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
  }
  unsigned long long tot;
  block_incl_scan_u64<NT>(dA, wsum, &tot);
  if (tid == 0) {
    admitted[inst] = adm;
    const long long a = ld_ll(&S.A[inst]) + (long long)tot;
    S.A[inst] = a;
    S.Aevt[inst] = a;
  }
}

template <int NT, int EM>
__global__ void __launch_bounds__(NT) pf_admit_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                       const long long* budget, const uint32_t* n_active,
                                                       const unsigned long long* k0,
                                                       const unsigned long long* A,
                                                       const unsigned long long* C, const uint32_t* cnt,
                                                       uint32_t* order, uint32_t* keyout, uint32_t* grant,
                                                       uint32_t* admitted, uint32_t* gslot) {
  extern __shared__ __align__(16) unsigned long long pf_sm[];
  unsigned long long* sbuf = pf_sm;              // [2 * PF_SCAP] the prefix + exchange buffer
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[NT / 32];
  __shared__ unsigned long long freed;
  __shared__ uint32_t m_s;
  const int tid = threadIdx.x;
  const uint32_t MA = S.MA;
  const long long B = budget[0];
  const uint32_t target = pf_target(B, n_active[0]);
  const uint32_t nA = cnt[0], nC = cnt[1];
  // ---- the first `target` entries of the order: A, plus the smallest of C
  for (uint32_t i = tid; i < nA; i += NT) sbuf[i] = A[i];
  if (tid == 0) m_s = nA;
  const uint32_t needC = target > nA ? target - nA : 0u;
  if (needC > 0 && nA + nC <= PF_SCAP) {
    // the whole crossing bucket fits beside A: sort them all, keep `target`
    for (uint32_t i = tid; i < nC; i += NT) sbuf[nA + i] = C[i];
    if (tid == 0) m_s = nA + nC;
  } else if (needC > 0) {
    // large crossing bucket: select its (target - |A|) smallest in place
    const unsigned long long* cb = C;
    __syncthreads();
    wselect<NT>(sel, nC, needC, 64, [&](uint32_t i, uint64_t& key, uint32_t& w) {
      key = cb[i]; w = 1u; return true; });
    const unsigned long long tau = sel.r.found ? sel.r.k : ~0ull;
    for (uint32_t i = tid; i < nC; i += NT) {
      const unsigned long long x = cb[i];
      if (x <= tau) sbuf[atomicAdd(&m_s, 1u)] = x;
    }
  }
  __syncthreads();
  const uint32_t mt = m_s;  // >= target entries, the first `target` of the order among them
  pf_finish<NT, EM>(S, cfg, cap, now, 0, 0, k0, sbuf, sbuf + PF_SCAP, mt, target, B, order, keyout,
                    grant, admitted, gslot, sel, wsum, freed);
}


// Prefix step of a multi-instance handle: one CTA per instance keeps the
// instance's packed words in shared memory, selects its first min(B, n)
// order entries by a count-weighted radix select, then pf_finish.
template <int NT, int EM>
__global__ void __launch_bounds__(NT) pf_multi_kernel(Slots S, augsched_config cfg, int64_t cap, uint64_t now,
                                                       long long* budget, uint32_t* n_active, uint32_t* order,
                                                       uint32_t* keyout, uint32_t* grant, uint32_t* admitted,
                                                       uint32_t* gslot, uint32_t sbuf_cap) {
  extern __shared__ __align__(16) unsigned long long pf_sm[];
  const uint32_t MA = S.MA;
  unsigned long long* kbuf = pf_sm;             // [MA] packed words of the instance
  unsigned long long* sbuf = pf_sm + MA;        // [sbuf_cap] the prefix
  unsigned long long* xch = sbuf + sbuf_cap;    // [sbuf_cap] sort exchange buffer
  __shared__ SelShm sel;
  __shared__ unsigned long long wsum[NT / 32];
  __shared__ unsigned long long freed;
  __shared__ uint32_t m_s;
  __shared__ long long B_s;
  const int tid = threadIdx.x;
  const uint32_t inst = blockIdx.x;
  const size_t base = (size_t)inst * MA;
  const Coef& k = S.coef[inst];
  const augsched_instance_params& ip = S.ip[inst];
  if (tid == 0) {
    B_s = token_limit(cfg, k, ip, cap, ld_ll(&S.A[inst]), ld_ll(&S.P[inst]));
    budget[inst] = B_s;
    m_s = 0;
  }
  unsigned long long myq = 0;
  for (uint32_t x = tid; x < MA; x += NT) {
    const uint32_t stv = S.st[base + x] & 15;
    const uint32_t tier = (stv >= ST_RUN && stv <= ST_WAIT) ? stv - ST_RUN : 3u;
    const uint32_t key = tier < 3 ? rank_key(k, ip, S.V[base + x], now, S.last[base + x], x) : 0u;
    kbuf[x] = ((unsigned long long)tier << PK_TIER) | ((unsigned long long)key << PK_KEY) | x;
    myq += tier < 3;
  }
  unsigned long long nq;
  block_incl_scan_u64<NT>(myq, wsum, &nq);   // syncs
  const long long B = B_s;
  const uint32_t target = pf_target(B, (uint32_t)nq);
  if (tid == 0) n_active[inst] = (uint32_t)nq;
  if (target > 0) {
    wselect<NT>(sel, MA, target, 64, [&](uint32_t i, uint64_t& key, uint32_t& w) {
      key = kbuf[i]; w = 1u; return (key >> PK_TIER) < 3; });
    const unsigned long long tau = sel.r.found ? sel.r.k : ~0ull;
    for (uint32_t x = tid; x < MA; x += NT) {
      const unsigned long long kx = kbuf[x];
      if ((kx >> PK_TIER) < 3 && kx <= tau) sbuf[atomicAdd(&m_s, 1u)] = kx;
    }
  }
  __syncthreads();
  pf_finish<NT, EM>(S, cfg, cap, now, inst, base, kbuf, sbuf, xch, m_s, target, B, order, keyout, grant,
                    admitted, gslot, sel, wsum, freed);
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

Slots slots_of(StepState& st, const augsched_instance_params* d_ip) {
  return Slots{st.st, st.V, st.last, st.ctx, st.kv, st.cpu, st.pend, st.A, st.P, st.Aevt, st.Asnap,
               st.coef, d_ip, st.max_active};
}

}  // namespace

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
  const size_t zwords = (size_t)n_inst + STEP_HIST_WORDS + STEP_MAX_PASS + 8;
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
      (rc = salloc(st, &st.gslot, N)))
    return rc;
  // one memset per step clears the queue counts, histograms and tile counters
  st.zwords = zwords;
  st.n_active = st.zbuf;
  st.ghist = st.zbuf + n_inst;
  st.tile_ctr = st.ghist + STEP_HIST_WORDS;
  st.pf_cnt = st.tile_ctr + STEP_MAX_PASS;
  cudaMemsetAsync(st.gslot, 0, sizeof(uint32_t) * N, s);
  cudaMemsetAsync(st.st, 0, sizeof(uint32_t) * N, s);
  cudaMemsetAsync(st.ctx, 0, sizeof(int32_t) * N, s);
  cudaMemsetAsync(st.kv, 0, sizeof(int32_t) * N, s);
  cudaMemsetAsync(st.cpu, 0, sizeof(int32_t) * N, s);
  cudaMemsetAsync(st.pend, 0, sizeof(int32_t) * N, s);
  cudaMemsetAsync(st.A, 0, sizeof(long long) * n_inst, s);
  cudaMemsetAsync(st.P, 0, sizeof(long long) * n_inst, s);
  cudaMemsetAsync(st.Aevt, 0, sizeof(long long) * n_inst, s);
  cudaMemsetAsync(st.lb_status, 0, sizeof(unsigned long long) * ((size_t)st.n_tiles << STEP_RB_MAX), s);
  cudaMemsetAsync(st.lb_gstatus, 0, sizeof(unsigned long long) * ((size_t)st.n_tiles << STEP_RB_MAX), s);
  st.G = 1;
  while ((uint64_t)st.G * st.G < st.n_tiles) ++st.G;   // ~sqrt(tiles) tiles per look-back group
  coef_kernel<<<(n_inst + 255) / 256, 256, 0, s>>>(cfg, d_ip, st.coef, n_inst);
  *launches += 1;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(pf_admit_kernel<PNT, PF_SCAP / PNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(unsigned long long) * 2 * PF_SCAP));
  cudaFuncSetAttribute(pf_multi_kernel<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PF_MULTI_SMEM);
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
                                                 st.max_active, d_err);
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
void run_records(StepState& st, const Slots& S, uint32_t* d_err, uint64_t now, cudaStream_t s,
                 uint64_t* launches) {
  if (!st.r_n) return;
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

static size_t pf_smem_bytes() { return sizeof(unsigned long long) * 2 * PF_SCAP; }

int step_run_prefix(StepState& st, const augsched_config& cfg, int64_t cap,
                    const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
                    augsched_step_out* out, cudaStream_t s, uint64_t* launches) {
  // the prefix selection is bounded by PF_SCAP; several instances need their
  // slots on chip (one CTA per instance)
  uint32_t scap = 32;
  while (scap < st.max_limit) scap <<= 1;
  const size_t msmem = sizeof(unsigned long long) * ((size_t)st.max_active + 2 * (size_t)scap);
  if (st.max_limit > PF_SCAP || (st.n_inst > 1 && msmem > PF_MULTI_SMEM))
    return step_run(st, cfg, cap, d_ip, d_err, now, out, s, launches);
  Slots S = slots_of(st, d_ip);
  run_records(st, S, d_err, now, s, launches);
  if (st.n_inst > 1) {
    if (scap <= 4 * 256)   // small limits: 256-thread CTAs, more instances resident per SM
      pf_multi_kernel<256, 4><<<st.n_inst, 256, msmem, s>>>(S, cfg, cap, now, st.budget, st.n_active, st.order,
                                                             st.key, st.grant, st.admitted, st.gslot, scap);
    else
      pf_multi_kernel<PNT, PF_SCAP / PNT><<<st.n_inst, PNT, msmem, s>>>(S, cfg, cap, now, st.budget, st.n_active,
                                                                        st.order, st.key, st.grant, st.admitted,
                                                                        st.gslot, scap);
    *launches += 1;
    out->budget = reinterpret_cast<const int64_t*>(st.budget);
    out->n_active = st.n_active;
    out->admitted = st.admitted;
    out->order = st.order;
    out->grant = st.grant;
    out->key = st.key;
    return cuda_check(cudaGetLastError(), "step_prefix");
  }
  cudaMemsetAsync(st.zbuf, 0, sizeof(uint32_t) * st.zwords, s);
  KeyArgs ka;
  ka.S = S; ka.cfg = cfg; ka.cap = cap; ka.now = now; ka.k0 = st.k0;
  ka.ghist = st.ghist; ka.n_active = st.n_active; ka.budget = st.budget; ka.npass = 1;
  ka.passes[0] = PassDesc{0, 64 - PF_BITS, PF_BITS, 0};
  ka.N = (uint32_t)st.N;
  ka.pf_cnt = st.pf_cnt;
  const size_t kblocks = (st.N + KNT * KU - 1) / (KNT * KU);
  const size_t kmax = (size_t)st.sms * AUGSCHED_KEYS_GRIDMUL;
  const int kgrid = (int)(kblocks < kmax ? kblocks : kmax);
  keys_kernel<<<kgrid, KNT, 0, s>>>(ka);
  pf_collect_kernel<<<kgrid, KNT, 0, s>>>(st.k0, (uint32_t)st.N, st.pf_cnt, st.pf_A, st.pf_C);
  pf_admit_kernel<PNT, PF_SCAP / PNT><<<1, PNT, pf_smem_bytes(), s>>>(S, cfg, cap, now, st.budget, st.n_active,
                                                                      st.k0, st.pf_A, st.pf_C, st.pf_cnt,
                                                                      st.order, st.key, st.grant, st.admitted,
                                                                      st.gslot);
  *launches += 3;
  out->budget = reinterpret_cast<const int64_t*>(st.budget);
  out->n_active = st.n_active;
  out->admitted = st.admitted;
  out->order = st.order;
  out->grant = st.grant;
  out->key = st.key;
  return cuda_check(cudaGetLastError(), "step_prefix");
}

int step_run(StepState& st, const augsched_config& cfg, int64_t cap,
             const augsched_instance_params* d_ip, uint32_t* d_err, uint64_t now,
             augsched_step_out* out, cudaStream_t s, uint64_t* launches) {
  Slots S = slots_of(st, d_ip);
  const uint32_t ni = st.n_inst;
  run_records(st, S, d_err, now, s, launches);
  cudaMemsetAsync(st.zbuf, 0, sizeof(uint32_t) * st.zwords, s);
  KeyArgs ka;
  ka.S = S; ka.cfg = cfg; ka.cap = cap; ka.now = now; ka.k0 = st.k0;
  ka.ghist = st.ghist; ka.n_active = st.n_active; ka.budget = st.budget; ka.npass = st.npass;
  for (int p = 0; p < st.npass; ++p) ka.passes[p] = st.passes[p];
  ka.N = (uint32_t)st.N;
  ka.pf_cnt = nullptr;
  const size_t kblocks = (st.N + KNT * KU - 1) / (KNT * KU);
  const int kgrid = (int)(kblocks < (size_t)st.sms * 8 ? kblocks : (size_t)st.sms * 8);
  keys_kernel<<<kgrid, KNT, 0, s>>>(ka);
  *launches += 1;
  unsigned long long *kin = st.k0, *kout = st.k1;
  for (int p = 0; p < st.npass; ++p) {
    SortArgs sa;
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
  admit_kernel<<<ni, ANT, 0, s>>>(S, cfg, cap, now, st.budget, st.n_active, st.order, st.grant,
                                  st.admitted);
  *launches += 1;
  out->budget = reinterpret_cast<const int64_t*>(st.budget);
  out->n_active = st.n_active;
  out->admitted = st.admitted;
  out->order = st.order;
  out->grant = st.grant;
  out->key = st.key;
  return cuda_check(cudaGetLastError(), "step");
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
