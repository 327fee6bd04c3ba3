// augsched_simulate: persistent per-instance simulation kernel for sm_100a.
// See sim.cuh for the design; the per-step sequence follows DESIGN.md §"Step
// sequence" (S1..S12), i.e. Algorithm 1 plus the engine model.
//
// The queue of an instance is held as two lists: R (running u swapped, tiers
// 0 and 1 of P:1221) and W (waiting_resume u waiting_new, tier 2, R16).  The
// order is (tier, key, id), so every R entry precedes every W entry and a
// step only needs the keys of the tier where the admission prefix ends:
//   - R keys are always computed (R is small: what fits in KV memory);
//   - W keys are computed only when the prefix reaches W, and then only the
//     smallest few matter: each lane keeps its two smallest W keys and the
//     block pops the global minimum round by round (one barrier per round)
//     until the popped demand reaches the limit;
//   - the grant / engine-advance loop touches R and the popped W entries only.
#include <cuda_runtime.h>
#include "sim.cuh"
#include "select.cuh"

namespace augsched {

constexpr int MAXPOP = 32;   // pop rounds before falling back to a radix select over W
#ifndef AUGSCHED_SIM_WPREFETCH
#define AUGSCHED_SIM_WPREFETCH 1
#endif
#ifndef AUGSCHED_SIM_RKSPEC
#define AUGSCHED_SIM_RKSPEC 1
#endif

#ifdef AUGSCHED_SIM_STATS
// Path counters and phase clocks of the stats build (tools/sim_stats.py).
__device__ unsigned long long g_sim_stats[64];
#define SSTAT(i, v) do { if ((threadIdx.x % SIM_NT) == 0) atomicAdd(&g_sim_stats[i], (unsigned long long)(v)); } while (0)
#define PT(i) do { if ((threadIdx.x % SIM_NT) == 0) s.pt[i] = clock64(); } while (0)
#else
#define SSTAT(i, v) do { } while (0)
#define PT(i) do { } while (0)
#endif

struct __align__(16) SimShm {
  union {
    SelBinsT<SIM_RB> b;              // radix-select histograms (fallback path)
    CandShmT<SIM_CAND> c;            // small candidate lists (fast path)
  } u;
  SelRes res;
  unsigned long long tw[3];          // per-tier demand of the step (unclamped)
  unsigned long long w2;             // demand total of the W list (maintained incrementally)
  unsigned int tc[3];                // per-tier candidate counts of the step
  unsigned long long rk[2][SIM_NW];  // pop rounds: per-warp smallest key, its demand and
  unsigned int rw[2][SIM_NW];        //   W position (double-buffered by round parity)
  unsigned int rp[2][SIM_NW];
  unsigned long long pk[MAXPOP];     // popped W entries of the step: key (| KEVICT if
  unsigned int pw[MAXPOP];           //   its grant was cancelled), demand, W position
  unsigned int pp[MAXPOP];
  unsigned int npop;
  int wmode;                         // which W entries the step grants (see WMODE_*)
  int wkeys;                         // W keys materialised in kscr[nR ..]
  int due;                           // intake or idle handling needed this iteration
  unsigned long long cnt[AUGSCHED_R_NFIELD];
  unsigned int c32[AUGSCHED_R_NFIELD];  // this call's counts (native 32-bit shared atomics),
                                        // folded into cnt when the instance's window ends
  unsigned int holes[2][HOLE_CAP];   // hole positions of R (0) and W (1)
  unsigned int nholes[2];
  unsigned int wtot[SIM_NW + 1];
  Coef coef;                         // per-instance constants (§8(c).1)
  augsched_instance_params ip;
  // instance scalars
  unsigned long long t, tT, min_ret, next_tick;
  long long A, P, A_snap, B;
  unsigned long long freed;
  unsigned int next_arr, n_r, n_w, n_pz, n_fin, wpos;
  unsigned int inst;
  unsigned int trace, r0, n;         // the instance's trace and its request range
  int run, idle, abort;
#ifdef AUGSCHED_SIM_STATS
  long long pt[9];                   // stats build: clock at the step's phase points
  int full;                          //   the step ran to its end
#endif
};

enum : int {
  WMODE_NONE = 0,   // the prefix ends in R (or B <= 0): no W entry is granted
  WMODE_POP = 1,    // the popped W entries s.pk/pw/pp are granted
  WMODE_ALL = 2,    // everything fits: every W entry is granted in full
  WMODE_KEY = 3,    // fallback: W keys materialised, grant by the key rule
};

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t INVALID = 0xffffffffu;

// Thread index within the instance's group, and the group barrier: the CTA
// when it runs one instance, the warp when it runs several.
#define ITID (threadIdx.x % SIM_NT)
__device__ __forceinline__ void ISYNC() {
  if (SIM_WPC > 1) __syncwarp();
  else __syncthreads();
}
// Phase fences (SIM_WPC > 1 and AUGSCHED_SIM_PSYNC): every iteration passes
// SIM_PHASES CTA barriers at fixed points, so the CTA's warps also run the
// phases inside a step together; a warp that skips the rest of a step (idle
// jump, finished window, no instance) passes the remaining ones.
// Fence set (bit i = fence i): 0 after intake, 1 after the R keys, 2 after
// the selection, 3 after the engine advance, 4 after the resolution.
#ifndef AUGSCHED_SIM_PSYNC
#define AUGSCHED_SIM_PSYNC 24
#endif
constexpr int SIM_PHASES = SIM_WPC > 1 ? __builtin_popcount(AUGSCHED_SIM_PSYNC) : 0;
// Every phase fence is this one barrier instruction (not inlined), so warps
// that reach a fence from different places of the step -- a warp that
// skips the rest of its step passes its remaining fences in phase_rest --
// still meet at the same bar.sync.
__device__ __noinline__ void cta_fence() { __syncthreads(); }
template <int I>
__device__ __forceinline__ void phase_bar(int& nb) {
  if (SIM_WPC > 1 && ((AUGSCHED_SIM_PSYNC >> I) & 1)) { cta_fence(); ++nb; }
}
__device__ __forceinline__ void phase_rest(int& nb) {
  if (SIM_PHASES) for (; nb < SIM_PHASES; ++nb) cta_fence();
}
__device__ __forceinline__ int isync_count(bool x) {
  if (SIM_WPC > 1) { __syncwarp(); return __popc(__ballot_sync(FULL, x)); }
  return __syncthreads_count(x);
}

__device__ __forceinline__ void err_set(const SimParams& p, uint32_t bits) { atomicOr(p.err, bits); }

// Block-wide exclusive scan of a 0/1 flag; returns this thread's prefix and
// (in s.wtot[SIM_NW]) the block total.  Contains two __syncthreads.
__device__ __forceinline__ uint32_t block_flag_scan(SimShm& s, bool f) {
  const int lane = ITID & 31, warp = ITID >> 5;
  const unsigned b = __ballot_sync(FULL, f);
  if (lane == 0) s.wtot[warp] = __popc(b);
  ISYNC();
  if (ITID == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < SIM_NW; ++w) { uint32_t x = s.wtot[w]; s.wtot[w] = acc; acc += x; }
    s.wtot[SIM_NW] = acc;
  }
  ISYNC();
  return s.wtot[warp] + __popc(b & ((1u << lane) - 1));
}

// Count into this call's 32-bit counters.
__device__ __forceinline__ void cinc(SimShm& s, int f, uint32_t v = 1u) { atomicAdd(&s.c32[f], v); }

// Shared 64-bit accumulation by one warp: a plain update when the CTA is a
// single warp (no other writer), else an atomic.
__device__ __forceinline__ void warp_add64(unsigned long long* x, unsigned long long v) {
  if (SIM_NW == 1) *x += v;
  else atomicAdd(x, v);
}

// One queue list by position: the scoring record (V, last, id | tier << 30)
// as one 16-byte entry (a single vector load per entry and step) and the
// demand beside it (read only for the entries a step grants or offers).
struct List {
  QEnt* q;          // e == INVALID marks a hole
  uint32_t* dem;    // demand of the next grant (R17, R18)
  __device__ __forceinline__ void put(uint32_t pos, uint32_t e, double v, uint32_t l, uint32_t d) const {
    QEnt x;
    x.V = v; x.last = l; x.e = e;
    q[pos] = x;
    dem[pos] = d;
  }
};

struct Ctx {
  const SimParams& p;
  SimShm& s;
  const Coef& k;                        // in shared memory (keeps registers free)
  const augsched_instance_params& ip;   // in shared memory
  // arena slices of this instance
  ReqState* rs;
  List R, W;
  uint32_t* pz_id;
  uint64_t* ret;
  uint64_t* K;      // step keys: R at [0, nR), W (when materialised) at [nR, nR + nW)
  uint32_t* Ws;     // step weights, same layout
  uint64_t* K2;     // secondary selections
  uint32_t* W2;
  uint32_t r0, n, trace;
};

__device__ __forceinline__ uint32_t gen_total(const DevTrace& tr, uint32_t rid) {
  const uint32_t s0 = tr.seg_off[rid], ns = tr.n_seg[rid];
  uint32_t g = 0;
  for (uint32_t q = 0; q < ns; ++q) g += tr.gen_true[s0 + q];
  return g;
}

// Composite order key (tier, score key, id): unique, < 2^KBITS.
__device__ __forceinline__ uint64_t order_key(uint32_t e, uint32_t key) {
  return ((uint64_t)(e >> 30) << 48) | ((uint64_t)key << 16) | (e & 0xFFFF);
}

// S2: one returned call (Algorithm 1 lines 10-24).
__device__ void do_return(Ctx& c, uint32_t id) {
  const DevTrace& tr = c.p.tr;
  SimShm& s = c.s;
  const uint32_t rid = c.r0 + id;
  ReqState r = c.rs[id];
  const uint32_t m = r.meta;
  const uint32_t kk = meta_seg(m);
  const int pol = (int)meta_pol(m);
  const uint32_t s0 = tr.seg_off[rid];
  const uint32_t ns = meta_nseg(m);
  const int32_t ctx = r.ctx, kv = r.kv, cpu = r.cpu;
  const uint64_t R = tr.ret_len[s0 + kk];
  const uint64_t On = tr.gen_pred[s0 + kk + 1];
  const bool has_next = kk + 1 < ns - 1;
  const double An = has_next ? (double)tr.dur_pred[s0 + kk + 1] : 0.0;
  const double V = intake_stage2(c.k, c.ip.policy_mode, pol, (uint64_t)ctx, R, On, An, has_next,
                                 (uint64_t)s.A_snap);
  uint32_t st, tier;
  if (pol == POL_P) {
    st = ST_RUN; tier = 0;
    atomicAdd((unsigned long long*)&s.P, (unsigned long long)(-(long long)kv));
    atomicAdd((unsigned long long*)&s.A, (unsigned long long)(long long)kv);
  } else if (pol == POL_S) { st = ST_SWAP; tier = 1; }
  else { st = ST_WAIT; tier = 2; }
  r.pend = (int32_t)R;
  r.meta = make_meta(kk + 1, st, (uint32_t)pol, ns);
  r.left = tr.gen_true[s0 + kk + 1];
  c.rs[id] = r;
  cinc(s, AUGSCHED_R_RETURNS);
  const uint32_t dem = demand_of(ctx, kv, cpu, (int32_t)R, c.p.cfg.s_in);
  // last is not reset on return (R14)
  if (tier < 2) c.R.put(atomicAdd(&s.n_r, 1u), id | (tier << 30), V, r.lastc, dem);
  else {
    c.W.put(atomicAdd(&s.n_w, 1u), id | (2u << 30), V, r.lastc, dem);
    atomicAdd(&s.w2, (unsigned long long)dem);
  }
}

// S3: arrival of request `id` at W position `pos` (Algorithm 1 lines 2-9).
__device__ void do_arrival(Ctx& c, uint32_t id, uint32_t pos, uint64_t t) {
  const DevTrace& tr = c.p.tr;
  const uint32_t rid = c.r0 + id;
  const uint32_t s0 = tr.seg_off[rid];
  const uint64_t L = tr.l_pre[rid];
  const uint64_t O = tr.gen_pred[s0];
  const bool has_call = tr.n_seg[rid] > 1;
  const double A = has_call ? (double)tr.dur_pred[s0] : 0.0;
  const double V = intake_stage1(c.k, c.ip.policy_mode, L, O, A, has_call, (uint64_t)c.s.A_snap);
  const uint32_t ns = tr.n_seg[rid];
  if (ns == 0 || ns > 255) {   // meta holds 8 bits: stop this instance, report E_INVALID
    err_set(c.p, 4u);
    c.s.cnt[AUGSCHED_R_ERR] |= 4;
    c.s.abort = 1;
  }
  ReqState r;
  r.ctx = 0; r.kv = 0; r.cpu = 0; r.pend = (int32_t)L;
  r.meta = make_meta(0, ST_WAIT, POL_D, ns);
  r.ft = 0; r.lastc = 0;
  r.left = tr.gen_true[s0];
  c.rs[id] = r;
  c.W.put(pos, id | (2u << 30), V, (uint32_t)t, (uint32_t)L);   // R14, R31
  atomicAdd(&c.s.w2, (unsigned long long)L);
}

// Remove the entries of list `L` (0 = R, 1 = W) whose id is INVALID.
__device__ void compact_list(SimShm& s, const List& l, int L, unsigned int& n_ref) {
  const int tid = ITID;
  ISYNC();
  const uint32_t nh = s.nholes[L];
  if (nh == 0) return;
  ISYNC();   // every lane has read nholes before thread 0 clears it
  if (nh <= HOLE_CAP) {
    if (tid == 0) {
      const uint32_t n = n_ref, n_new = n - nh;
      uint32_t* h = s.holes[L];
      for (uint32_t a = 1; a < nh; ++a) {  // insertion sort (few holes)
        uint32_t x = h[a];
        int b = (int)a - 1;
        while (b >= 0 && h[b] > x) { h[b + 1] = h[b]; --b; }
        h[b + 1] = x;
      }
      int j = (int)nh - 1;
      int src = (int)n - 1;
      for (uint32_t a = 0; a < nh; ++a) {
        const uint32_t hp = h[a];
        if (hp >= n_new) break;
        while (j >= 0 && (int)h[j] == src) { --j; --src; }
        l.q[hp] = l.q[src];
        l.dem[hp] = l.dem[src];
        --src;
      }
      n_ref = n_new;
      s.nholes[L] = 0;
    }
    ISYNC();
    return;
  }
  // many removals: in-place tiled stream compaction
  if (tid == 0) s.wpos = 0;
  const uint32_t n = n_ref;
  for (uint32_t base = 0; base < n; base += SIM_NT) {
    const uint32_t i = base + tid;
    QEnt x;
    x.e = INVALID;
    uint32_t dem = 0;
    if (i < n) { x = l.q[i]; if (x.e != INVALID) dem = l.dem[i]; }
    const bool keep = x.e != INVALID;
    const uint32_t pre = block_flag_scan(s, keep);  // syncs: all reads of the tile are done
    if (keep) { l.q[s.wpos + pre] = x; l.dem[s.wpos + pre] = dem; }
    ISYNC();
    if (tid == 0) s.wpos += s.wtot[SIM_NW];
    ISYNC();
  }
  if (tid == 0) { n_ref = s.wpos; s.nholes[L] = 0; }
  ISYNC();
}

__device__ __forceinline__ void mark_hole(SimShm& s, int L, uint32_t pos) {
  const uint32_t h = atomicAdd(&s.nholes[L], 1u);
  if (h < HOLE_CAP) s.holes[L][h] = pos;
}

// Remove paused entries marked INVALID (small list; tiled compaction).
__device__ void compact_paused(Ctx& c) {
  SimShm& s = c.s;
  const int tid = ITID;
  ISYNC();
  if (tid == 0) s.wpos = 0;
  const uint32_t n = s.n_pz;
  for (uint32_t base = 0; base < n; base += SIM_NT) {
    const uint32_t i = base + tid;
    const uint32_t id = i < n ? c.pz_id[i] : INVALID;
    const bool keep = id != INVALID;
    const uint32_t pre = block_flag_scan(s, keep);
    if (keep) c.pz_id[s.wpos + pre] = id;
    ISYNC();
    if (tid == 0) s.wpos += s.wtot[SIM_NW];
    ISYNC();
  }
  if (tid == 0) s.n_pz = s.wpos;
  ISYNC();
}

// Selections, kept out of line: one instantiation of each serves every call
// site (the hot loop stays small in the instruction cache).
// Weighted radix select over arrays: key K[i] (or KMASK - K[i] when rev),
// weight W[i]; entries with weight 0 are skipped.
__device__ __noinline__ void select_arr(SimShm& s, const uint64_t* K, const uint32_t* W, uint32_t n,
                                        uint64_t D, int nbits, bool rev) {
  wselect<SIM_NT, SIM_RB>(s.u.b, s.res, n, D, nbits, [&](uint32_t i, uint64_t& key, uint32_t& w) {
    w = W[i];
    key = rev ? KMASK - K[i] : K[i];
    return w > 0;
  });
}

__device__ __noinline__ void select_cand(SimShm& s, int list, int m, uint64_t D, uint64_t w0) {
  rank_select<SIM_NT, SIM_CAND>(s.u.c, list, s.res, m, D, w0);
}

// Thread 0 prepares iteration s.t: stop rule, S1 snapshot, whether intake
// or the idle jump must run, and (when no intake is due) the token limit.
__device__ __noinline__ void prep_step(const SimParams& p, SimShm& s, uint32_t n) {
  s.run = (s.n_fin < n) && (s.t < p.max_iters) && !s.abort;
  s.tT = s.t * p.cfg.t_fwd_ticks;
  s.A_snap = s.A;
  s.due = s.n_r + s.n_w == 0 || s.tT >= s.min_ret || s.tT >= s.next_tick;
  if (!s.due) s.B = token_limit(p.cfg, s.coef, s.ip, p.cap, s.A, s.P);
  s.tw[0] = s.tw[1] = s.tw[2] = 0;
  s.tc[0] = s.tc[1] = s.tc[2] = 0;
  s.wkeys = 0;
}

// Order key of W entry i at iteration t (out of line: the rare rescans and
// materialisations share one copy).
__device__ __noinline__ uint64_t w_order_key(const SimShm& s, const QEnt* q, uint32_t i, uint64_t t) {
  const QEnt x = q[i];
  return order_key(x.e, rank_key(s.coef, s.ip, x.V, t, x.last, x.e & 0xFFFF));
}

// Grant rule of the step (R17): full demand before k*, the remainder at k*,
// nothing after it or for an entry whose grant was cancelled (KEVICT).
struct GrantRule {
  long long B;
  uint64_t kstar, wb;
  bool found;
  __device__ __forceinline__ uint32_t operator()(uint64_t Ki, uint32_t dem) const {
    if (Ki & KEVICT) return 0u;
    if (B <= 0) return 0u;
    if (!found || Ki < kstar) return dem;
    if (Ki == kstar) return (uint32_t)((uint64_t)B - wb);
    return 0u;
  }
};

// Start (or resume) instance `inst` on this warp group: constants, trace
// bounds, the resumable header, this window's counters.  False when the
// instance cannot run (its trace exceeds the arena; reported in its record).
__device__ bool inst_begin(const SimParams& p, SimShm& s, uint32_t inst) {
  const int tid = ITID;
  const size_t off = (size_t)inst * p.max_active;
  const Arena& a = p.ar;
  if (tid == 0) { s.coef = make_coef(p.cfg, p.ip[inst]); s.ip = p.ip[inst]; }
  ISYNC();
  Ctx c{p, s, s.coef, s.ip, a.rs + off,
        List{a.r_q + off, a.r_dem + off},
        List{a.w_q + off, a.w_dem + off},
        a.pz_id + off, a.ret + off, a.kscr + off, a.wscr + off, a.kscr2 + off, a.wscr2 + off, 0, 0, 0};
  c.trace = p.inst_trace[inst];
  c.r0 = p.tr.req_off[c.trace];
  c.n = p.tr.req_off[c.trace + 1] - c.r0;
  if (tid == 0) { s.inst = inst; s.trace = c.trace; s.r0 = c.r0; s.n = c.n; }
  const uint32_t n = c.n;
  InstHdr& H = p.hdr[inst];
  augsched_result& acc = p.acc[inst];
  if (n > p.max_active) {  // trace longer than the arena
    if (tid == 0) { err_set(p, 2u); acc.f[AUGSCHED_R_ERR] |= 2; }
    ISYNC();
    if (tid == 0) p.out[inst] = acc;
    return false;
  }
  // ---- load (or initialise) the resumable state -------------------------
  if (tid == 0) {
    if (!H.started) {
      H.t = 0; H.A = 0; H.P = 0; H.min_ret = ~0ull; H.next_arr = 0; H.n_r = 0; H.n_w = 0; H.n_pz = 0;
      H.w2 = 0;
      H.n_fin = 0; H.started = 1;
    }
    s.t = H.t; s.A = H.A; s.P = H.P; s.min_ret = H.min_ret; s.next_arr = H.next_arr;
    s.n_r = H.n_r; s.n_w = H.n_w; s.n_pz = H.n_pz; s.n_fin = H.n_fin; s.w2 = H.w2;
    s.nholes[0] = s.nholes[1] = 0;
    s.abort = 0;
    s.next_tick = s.next_arr < n ? p.tr.arr_tick[c.r0 + s.next_arr] : ~0ull;
  }
  for (int f = tid; f < AUGSCHED_R_NFIELD; f += SIM_NT) { s.cnt[f] = acc.f[f]; s.c32[f] = 0; }
  ISYNC();
  if (tid == 0) s.cnt[AUGSCHED_R_NREQ] = n;
  if (tid == 0) prep_step(p, s, n);
  ISYNC();
  return true;
}

// One iteration of the instance (Algorithm 1 + engine model).  False when
// the instance's window is over (all requests finished, max_iters reached,
// or aborted).
__device__ bool inst_step(const SimParams& p, SimShm& s) {
  int nb = 0;
#ifdef AUGSCHED_SIM_STATS
  if (ITID == 0) s.full = 0;
#endif
  PT(0);
  if (!s.run) { phase_rest(nb); return false; }
  const int tid = ITID;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t inst = s.inst;
  const size_t off = (size_t)inst * p.max_active;
  const Arena& a = p.ar;
  Ctx c{p, s, s.coef, s.ip, a.rs + off,
        List{a.r_q + off, a.r_dem + off},
        List{a.w_q + off, a.w_dem + off},
        a.pz_id + off, a.ret + off, a.kscr + off, a.wscr + off, a.kscr2 + off, a.wscr2 + off, 0, 0, 0};
  c.trace = s.trace;
  c.r0 = s.r0;
  c.n = s.n;
  const uint64_t T = p.cfg.t_fwd_ticks;
  const uint32_t n = c.n;
  augsched_result& acc = p.acc[inst];
  const int64_t cap = p.cap;
  auto key_of = [&](double V, uint64_t t, uint32_t last, uint32_t e) -> uint32_t {
    return rank_key(c.k, c.ip, V, t, last, e & 0xFFFF);
  };
  (void)lane; (void)warp; (void)acc;
  const uint64_t t = s.t, tT = s.tT;
  if (s.due) {
    // ---- S2 returns --------------------------------------------------------
    if (tT >= s.min_ret) {
      const uint32_t npz = s.n_pz;
      unsigned long long mr = ~0ull;   // the next return among the calls still out
      for (uint32_t i = tid; i < npz; i += SIM_NT) {
        const uint32_t id = c.pz_id[i];
        const uint64_t rt = c.ret[id];
        if (rt <= tT) { do_return(c, id); c.pz_id[i] = INVALID; }
        else mr = rt < mr ? rt : mr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, mr, o);
        mr = y < mr ? y : mr;
      }
      ISYNC();   // every lane has read min_ret
      if (tid == 0) s.min_ret = ~0ull;
      ISYNC();
      if ((tid & 31) == 0) atomicMin(&s.min_ret, mr);
      compact_paused(c);   // syncs
    }
    // ---- S3 arrivals (ticks are sorted: the arrivals are a prefix) ----------
    if (tT >= s.next_tick) for (;;) {
      const uint32_t j = s.next_arr + tid;
      const bool arrive = j < n && p.tr.arr_tick[c.r0 + j] <= tT;
      const int cnt = isync_count(arrive);
      if (arrive) do_arrival(c, j, s.n_w + tid, t);
      ISYNC();
      if (tid == 0) {
        s.n_w += cnt; s.next_arr += cnt; s.cnt[AUGSCHED_R_ARRIVED] += cnt;
        if (cnt < SIM_NT) s.next_tick = s.next_arr < n ? p.tr.arr_tick[c.r0 + s.next_arr] : ~0ull;
      }
      ISYNC();
      if (cnt < SIM_NT) break;
    }
    // ---- idle jump (not counted) or S4 token limit ---------------------------
    ISYNC();   // every lane has read t / tT / run before thread 0 may move them
    if (tid == 0) {
      s.idle = 0;
      if (s.n_r + s.n_w == 0) {
        uint64_t te = ~0ull;
        if (s.next_arr < n) te = (p.tr.arr_tick[c.r0 + s.next_arr] + T - 1) / T;
        if (s.n_pz > 0) { const uint64_t tr_ = (s.min_ret + T - 1) / T; te = tr_ < te ? tr_ : te; }
        if (te == ~0ull) { s.idle = 2; s.run = 0; }
        else { s.t = te; s.idle = 1; prep_step(p, s, n); }
      } else {
        s.B = token_limit(p.cfg, c.k, c.ip, cap, s.A, s.P);
      }
    }
    ISYNC();
    if (s.idle) { phase_rest(nb); return true; }
  }
  PT(1);
  phase_bar<0>(nb);
  const uint32_t nR = s.n_r, nW = s.n_w, na = nR + nW;
  const long long B = s.B;
  const unsigned long long Bu = B > 0 ? (unsigned long long)B : 0ull;
  const unsigned lt = (1u << lane) - 1;
  // ---- S5 keys of R, per-tier demand, running / swapped candidate lists ----
  {
    unsigned long long tw0 = 0, tw1 = 0;
    for (uint32_t b0 = 0; b0 < nR; b0 += SIM_NT) {   // warp-uniform trip count
      const uint32_t i = b0 + tid;
      uint32_t tier = 3, d = 0;
      uint64_t Ki = 0;
      if (i < nR) {
        const QEnt x = c.R.q[i];
        d = c.R.dem[i];
        tier = x.e >> 30;
        Ki = order_key(x.e, key_of(x.V, t, x.last, x.e));
        c.K[i] = Ki;
        c.Ws[i] = d;
        if (tier == 0) tw0 += d; else tw1 += d;
      }
#pragma unroll
      for (uint32_t tt = 0; tt < 2; ++tt) {
        const unsigned m = __ballot_sync(FULL, tier == tt);
        if (m) {
          const int leader = __ffs(m) - 1;
          uint32_t q0 = 0;
          if (lane == leader) q0 = atomicAdd(&s.tc[tt], (unsigned)__popc(m));
          q0 = __shfl_sync(FULL, q0, leader);
          const uint32_t q = q0 + __popc(m & lt);
          if (tier == tt && q < SIM_CAND) { s.u.c.ck[tt][q] = Ki; s.u.c.cw[tt][q] = d; }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tw0 += __shfl_xor_sync(FULL, tw0, o);
      tw1 += __shfl_xor_sync(FULL, tw1, o);
    }
    if (lane == 0) {
      if (tw0) warp_add64(&s.tw[0], tw0);
      if (tw1) warp_add64(&s.tw[1], tw1);
    }
    if (tid == 0) {
      s.cnt[AUGSCHED_R_BUSY_STEPS] += 1;
      s.cnt[AUGSCHED_R_DECISIONS] += na;
      if (na > s.cnt[AUGSCHED_R_MAXQ]) s.cnt[AUGSCHED_R_MAXQ] = na;
    }
  }
  ISYNC();
  PT(2);
  phase_bar<1>(nb);
  // ---- S6/S7 order + admission: the last admitted entry k* ------------------
  // Tiers are ordered running < swapped < waiting, so the tier where the
  // prefix ends follows from the per-tier totals.
  {
    const unsigned long long w0 = s.tw[0], w1 = s.tw[1];
    int wmode = WMODE_NONE;
    SSTAT(18, 1);
    SSTAT(30, nR);
    SSTAT(31, nW);
    if (B <= 0) {
      if (tid == 0) { s.res.found = 1; s.res.k = 0; s.res.wbelow = 0; }  // nothing admitted
    } else if (w0 >= Bu) {
      SSTAT(17, 1);
      SSTAT(25, s.tc[0]);
      if (s.tc[0] <= SIM_CAND) { SSTAT(23, 1); select_cand(s, 0, (int)s.tc[0], Bu, 0); }
      else { SSTAT(24, 1); select_arr(s, c.K, c.Ws, nR, Bu, KBITS, false); }
    } else if (w0 + w1 >= Bu) {
      SSTAT(22, 1);
      if (s.tc[1] <= SIM_CAND) { SSTAT(23, 1); select_cand(s, 1, (int)s.tc[1], Bu, w0); }
      else { SSTAT(24, 1); select_arr(s, c.K, c.Ws, nR, Bu, KBITS, false); }
    } else {
      // the prefix reaches W.  The W demand total is maintained
      // incrementally; when everything fits no W key is needed.
      const unsigned long long wall = w0 + w1 + s.w2;
      SSTAT(0, 1);
      if (wall < Bu) {
        SSTAT(16, 1);
        if (tid == 0) { s.res.found = 0; s.res.total = wall; }   // everything admitted
        wmode = WMODE_ALL;
      } else {
#if AUGSCHED_SIM_WPREFETCH
        // the W list's lines to L2 first (non-blocking), so the scan's rounds
        // of dependent loads after the first find them on chip
        {
          const uint32_t nb = nW * (uint32_t)sizeof(QEnt);
          const char* wb = reinterpret_cast<const char*>(c.W.q);
          for (uint32_t o = (uint32_t)tid * 128u; o < nb; o += 128u * SIM_NT)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wb + o));
        }
#endif
        // one pass over W: this lane's two smallest keys and their positions
        // (one 16-byte load per entry), then their demands
        uint64_t c1 = ~0ull, c2 = ~0ull;
        uint32_t cp1 = 0, cp2 = 0;
        constexpr int U = SIM_UNROLL;  // entries in flight per thread (independent L2 loads)
        auto wscan = [&](auto keyf) {
          for (uint32_t b0 = 0; b0 < nW; b0 += SIM_NT * U) {
            QEnt x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t i = b0 + u * SIM_NT + tid;
              if (i < nW) x[u] = c.W.q[i];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t i = b0 + u * SIM_NT + tid;
              if (i < nW) {
                const uint64_t Ki = order_key(x[u].e, keyf(x[u]));
                if (Ki < c2) {
                  if (Ki < c1) { c2 = c1; cp2 = cp1; c1 = Ki; cp1 = i; }
                  else { c2 = Ki; cp2 = i; }
                }
              }
            }
          }
        };
#if AUGSCHED_SIM_RKSPEC
        if (c.ip.ranking == AUGSCHED_RANK_AUGSERVE) {
          // the value ranking (R3) with its constants in registers: the same
          // operations as sched_key
          const double al = c.k.alpha, Ts = c.k.Ts;
          wscan([&](const QEnt& x) {
            const double s_ = dsub(x.V, dmul(al, dmul(u2d(t - x.last), Ts)));
            const uint32_t u_ = __float_as_uint(__double2float_rn(s_));
            return (u_ & 0x80000000u) ? ~u_ : (u_ | 0x80000000u);
          });
        } else
#endif
          wscan([&](const QEnt& x) { return key_of(x.V, t, x.last, x.e); });
        const uint32_t cw1 = c1 != ~0ull ? c.W.dem[cp1] : 0u;
        const uint32_t cw2 = c2 != ~0ull ? c.W.dem[cp2] : 0u;
        // pop the smallest remaining W keys in order, one per round (one
        // barrier each); a lane offers c1, then c2, then rescans its own
        // positions for the next key above the last one popped
        unsigned long long wb = w0 + w1;
        uint64_t myk = c1;
        uint32_t myw = cw1, myp = cp1;
        int cons = 0;
        for (int r = 0; r < MAXPOP; ++r) {
          uint64_t mk = myk;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(FULL, mk, o);
            mk = y < mk ? y : mk;
          }
          const unsigned own = __ballot_sync(FULL, myk == mk);
          if (lane == __ffs(own) - 1) { s.rk[r & 1][warp] = mk; s.rw[r & 1][warp] = myw; s.rp[r & 1][warp] = myp; }
          ISYNC();
          uint64_t bk = s.rk[r & 1][0];
          uint32_t bw = s.rw[r & 1][0], bp = s.rp[r & 1][0];
#pragma unroll
          for (int w = 1; w < SIM_NW; ++w) {
            const uint64_t x = s.rk[r & 1][w];
            if (x < bk) { bk = x; bw = s.rw[r & 1][w]; bp = s.rp[r & 1][w]; }
          }
          if (bk == ~0ull) break;  // not reachable: the W total reaches B
          if (tid == 0) { s.pk[r] = bk; s.pw[r] = bw; s.pp[r] = bp; }
          SSTAT(27, 1);
          if (wb + bw >= Bu) {
            SSTAT(26, 1);
            if (tid == 0) { s.res.found = 1; s.res.k = bk; s.res.wbelow = wb; s.npop = r + 1; }
            wmode = WMODE_POP;
            break;
          }
          wb += bw;
          if (myk == bk) {
            if (++cons == 1) { myk = c2; myw = cw2; myp = cp2; }
            else {
              SSTAT(28, 1);
              uint64_t nk = ~0ull;
              uint32_t nw = 0, np = 0;
              for (uint32_t i = tid; i < nW; i += SIM_NT) {
                const uint64_t Ki = w_order_key(s, c.W.q, i, t);
                if (Ki > bk && Ki < nk) { nk = Ki; nw = c.W.dem[i]; np = i; }
              }
              myk = nk; myw = nw; myp = np;
            }
          }
        }
        if (wmode != WMODE_POP) {
          SSTAT(20, 1);
          // many small W demands: materialise every key and radix-select
          for (uint32_t i = tid; i < nW; i += SIM_NT) {
            c.K[nR + i] = w_order_key(s, c.W.q, i, t);
            c.Ws[nR + i] = c.W.dem[i];
          }
          if (tid == 0) s.wkeys = 1;
          select_arr(s, c.K, c.Ws, na, Bu, KBITS, false);
          wmode = WMODE_KEY;
        }
      }
    }
    if (tid == 0) s.wmode = wmode;
    ISYNC();
  }
  const int wmode = s.wmode;
  const bool found = s.res.found != 0;
  const GrantRule grant{B, B > 0 ? s.res.k : 0ull, s.res.wbelow, found};
  const long long need = B <= 0 ? 0 : (found ? B : (long long)s.res.total);
  long long freev = cap - s.A - s.P;
  // Granted entries are addressed by a virtual index v: v < nR is R entry v,
  // v >= nR is the (v - nR)-th W candidate: popped entry (WMODE_POP) or W
  // position (WMODE_ALL / WMODE_KEY).
  const uint32_t nGW = wmode == WMODE_POP ? s.npop : (wmode == WMODE_NONE ? 0u : nW);
  auto w_pos = [&](uint32_t j) -> uint32_t { return wmode == WMODE_POP ? s.pp[j] : j; };
  auto w_key = [&](uint32_t j) -> uint64_t {
    if (wmode == WMODE_POP) return s.pk[j];
    return s.wkeys ? c.K[nR + j] : 0ull;   // WMODE_ALL without resolution: every key passes
  };
  PT(3);
  phase_bar<2>(nb);
  // ---- S8 memory resolution (R20) -------------------------------------------
  if (need > freev) {
    SSTAT(29, 1);
    // (1) demote Preserve-paused contexts, kv desc, id asc
    const uint64_t D0 = (uint64_t)(need - freev);
    const uint32_t npz = s.n_pz;
    SSTAT(2, s.P == 0);
    SSTAT(3, npz);
    auto getp = [&](uint32_t i, uint64_t& key, uint32_t& w) {
      const uint32_t id = c.pz_id[i];
      const int32_t kv = c.rs[id].kv;
      if (meta_pol(c.rs[id].meta) != POL_P || kv <= 0) return false;
      key = ((uint64_t)(0xFFFFFFFFu - (uint32_t)kv) << 16) | id;
      w = (uint32_t)kv;
      return true;
    };
    if (tid == 0) { s.tc[0] = 0; s.freed = 0; }
    ISYNC();
    // P = the KV of the Preserve-paused requests: none to demote when it is 0
    // (88 % of the resolutions on the bench windows)
    if (s.P > 0) {
    for (uint32_t i = tid; i < npz; i += SIM_NT) {
      uint64_t key; uint32_t w;
      if (getp(i, key, w)) {
        const uint32_t q = atomicAdd(&s.tc[0], 1u);
        if (q < SIM_CAND) { s.u.c.ck[0][q] = key; s.u.c.cw[0][q] = w; }
      }
    }
    ISYNC();
    if (s.tc[0] <= SIM_CAND) select_cand(s, 0, (int)s.tc[0], D0, 0);
    else {
      // many Preserve-paused contexts: materialise (key, kv) and select over the arrays
      for (uint32_t i = tid; i < npz; i += SIM_NT) {
        uint64_t key = 0; uint32_t w = 0;
        if (!getp(i, key, w)) w = 0;
        c.K2[i] = key; c.W2[i] = w;
      }
      ISYNC();
      select_arr(s, c.K2, c.W2, npz, D0, 48, false);
    }
    {
      const bool f0 = s.res.found != 0;
      const uint64_t k0 = s.res.k;
      for (uint32_t i = tid; i < npz; i += SIM_NT) {
        uint64_t key; uint32_t w;
        if (getp(i, key, w) && (!f0 || key <= k0)) {
          const uint32_t id = c.pz_id[i];
          atomicAdd(&s.freed, (unsigned long long)w);
          c.rs[id].kv = 0;
          c.rs[id].meta = meta_with(c.rs[id].meta, meta_st(c.rs[id].meta), POL_D);
          cinc(s, AUGSCHED_R_DEMOTIONS);
        }
      }
    }
    }
    ISYNC();
    freev += (long long)s.freed;
    if (tid == 0) { s.P -= (long long)s.freed; s.tc[1] = 0; }
    if (need > freev && (wmode == WMODE_ALL) && !s.wkeys) {
      // the eviction order needs the W keys of this step
      ISYNC();
      for (uint32_t i = tid; i < nW; i += SIM_NT) c.K[nR + i] = w_order_key(s, c.W.q, i, t);
      if (tid == 0) s.wkeys = 1;
    }
    ISYNC();
    // (2) evict from the tail of the order over entries with kv + g > 0
    SSTAT(4, need > freev);
    if (need > freev) {
      const uint64_t D1 = (uint64_t)(need - freev);
      const uint32_t nv = nR + nGW;
      for (uint32_t v = tid; v < nv; v += SIM_NT) {
        uint64_t Ki;
        uint32_t w;
        if (v < nR) {
          Ki = c.K[v];
          w = (uint32_t)c.rs[c.R.q[v].e & 0xFFFF].kv + grant(Ki, c.R.dem[v]);
        } else {
          const uint32_t j = v - nR;
          Ki = w_key(j);
          w = grant(Ki, wmode == WMODE_POP ? s.pw[j] : c.W.dem[j]);   // W entries hold no KV
        }
        c.K2[v] = Ki;
        c.W2[v] = w;
        if (w > 0) {
          const uint32_t q = atomicAdd(&s.tc[1], 1u);
          if (q < SIM_CAND) { s.u.c.ck[1][q] = KMASK - Ki; s.u.c.cw[1][q] = w; }
        }
      }
      ISYNC();
      if (s.tc[1] <= SIM_CAND) select_cand(s, 1, (int)s.tc[1], D1, 0);
      else select_arr(s, c.K2, c.W2, nv, D1, KBITS, true);
      const bool f1 = s.res.found != 0;
      const uint64_t k1 = s.res.k;
      for (uint32_t v = tid; v < nv; v += SIM_NT) {
        const uint32_t w = c.W2[v];
        const uint64_t Ki = c.K2[v];
        if (w == 0 || (f1 && KMASK - Ki > k1)) continue;
        cinc(s, AUGSCHED_R_EVICTIONS);
        if (v < nR) {
          // running / swapped entry: drop its KV and requeue it in W
          const QEnt x = c.R.q[v];
          const uint32_t id = x.e & 0xFFFF;
          ReqState r = c.rs[id];
          atomicAdd((unsigned long long*)&s.A, (unsigned long long)(-(long long)r.kv));
          r.kv = 0;
          r.cpu = 0;
          r.meta = meta_with(r.meta, ST_WAIT, meta_pol(r.meta));
          c.rs[id] = r;
          const uint32_t nd = demand_of(r.ctx, 0, 0, r.pend, p.cfg.s_in);
          c.W.put(atomicAdd(&s.n_w, 1u), id | (2u << 30), x.V, x.last, nd);
          atomicAdd(&s.w2, (unsigned long long)nd);
          c.R.q[v].e = INVALID;
          c.K[v] |= KEVICT;
          mark_hole(s, 0, v);
        } else {
          // granted W entry: its grant is cancelled (it holds no KV)
          const uint32_t j = v - nR;
          if (wmode == WMODE_POP) s.pk[j] |= KEVICT;
          else c.K[nR + j] |= KEVICT;
        }
      }
      ISYNC();
    }
  }
  PT(4);
  phase_bar<4>(nb);
  PT(5);
  // ---- S9 last = t for granted entries; S10 engine advance -------------------
  {
    uint32_t my_tok = 0, my_adm = 0;
    long long accA = 0, accP = 0;
    unsigned long long accW2 = 0;   // demand leaving W
    const uint32_t nv = nR + nGW;
    for (uint32_t v = tid; v < nv; v += SIM_NT) {
      const bool inR = v < nR;
      uint32_t pos, e, dem;
      uint64_t Ki;
      if (inR) {
        pos = v;
        e = c.R.q[v].e;
        if (e == INVALID) continue;        // evicted to W this step
        Ki = c.K[v];
        dem = c.R.dem[v];
      } else {
        const uint32_t j = v - nR;
        pos = w_pos(j);
        e = c.W.q[pos].e;
        Ki = w_key(j);
        dem = wmode == WMODE_POP ? s.pw[j] : c.W.dem[pos];
      }
      const uint32_t g = grant(Ki, dem);
      if (g == 0) continue;
      my_tok += g; my_adm += 1;
      const uint32_t id = e & 0xFFFF;
      const uint32_t rid = c.r0 + id;
      ReqState r = c.rs[id];
      int32_t ctx = r.ctx, kv = r.kv, cpu = r.cpu, pend = r.pend;
      const int32_t kv_snap = kv;
      uint32_t m = r.meta;
      const uint32_t seg = meta_seg(m), pol = meta_pol(m);
      long long dA = 0, dP = 0;
      bool leave = false;
      if (cpu > 0) {                                   // swap-in
        cpu -= (int32_t)g; kv += (int32_t)g; dA += g;
      } else if ((ctx - kv) + pend > 0) {              // recompute, then prefill/assimilate
        const int32_t rc = (int32_t)g < ctx - kv ? (int32_t)g : ctx - kv;
        kv += rc;
        const int32_t pp = (int32_t)g - rc;
        pend -= pp; ctx += pp; kv += pp;
        dA += g;
      } else {                                         // decode one token
        ctx += 1; kv += 1; dA += 1;
        if (r.ft == 0) r.ft = (uint32_t)(t + 1);      // R22
        if (--r.left == 0) {                           // segment end
          leave = true;
          if (seg + 1 == meta_nseg(m)) {               // finish
            dA -= kv; kv = 0;
            m = meta_with(m, ST_DONE, pol);
            const uint64_t arr = p.tr.arr_tick[rid];
            const uint64_t fin = t + 1;
            const uint64_t ttft = (uint64_t)r.ft * T - arr;
            const uint64_t e2e = fin * T - arr;
            const uint64_t gt = gen_total(p.tr, rid);
            const bool ok = ttft < c.ip.slo_ttft_ticks &&
                            e2e * c.ip.slo_norm_den < (uint64_t)c.ip.slo_norm_num * T * gt;
            const bool ok5 = ttft < 5 * c.ip.slo_ttft_ticks &&
                             e2e * c.ip.slo_norm_den < 5 * (uint64_t)c.ip.slo_norm_num * T * gt;
            atomicAdd(&s.n_fin, 1u);
            cinc(s, AUGSCHED_R_COMPLETED);
            if (ok) cinc(s, AUGSCHED_R_SLO_OK);
            if (ok5) cinc(s, AUGSCHED_R_SLO_OK_5X);
            atomicMax(&s.c32[AUGSCHED_R_MAKESPAN], (uint32_t)fin);
            atomicAdd(&s.cnt[AUGSCHED_R_SUM_TTFT], (unsigned long long)ttft);
            atomicAdd(&s.cnt[AUGSCHED_R_SUM_E2E], (unsigned long long)e2e);
            atomicAdd(&s.cnt[AUGSCHED_R_SUM_GEN], (unsigned long long)gt);
            atomicAdd(&acc.hist_ttft[hist_bin(ttft)], 1u);   // rare: global atomics
            atomicAdd(&acc.hist_norm[hist_bin(e2e / gt)], 1u);
          } else {                                     // issue call `seg` (R13, R21)
            const uint32_t s0 = p.tr.seg_off[rid];
            const double Ti = (double)p.tr.dur_pred[s0 + seg];
            const int np = select_policy(c.k, (uint64_t)ctx, Ti,
                                         (uint64_t)(s.A_snap - (long long)kv_snap),
                                         c.ip.policy_mode);
            const uint64_t rt = (t + 1) * T + p.tr.dur_true[s0 + seg];
            c.ret[id] = rt;
            r.lastc = (uint32_t)t;
            dA -= kv;
            if (np == POL_P) { dP += kv; cinc(s, AUGSCHED_R_CALLS_PRESERVE); }
            else if (np == POL_S) { cpu = ctx; kv = 0; cinc(s, AUGSCHED_R_CALLS_SWAP); }
            else { kv = 0; cinc(s, AUGSCHED_R_CALLS_DISCARD); }
            m = meta_with(m, ST_PAUSED, (uint32_t)np);
            const uint32_t q = atomicAdd(&s.n_pz, 1u);
            c.pz_id[q] = id;
            atomicMin(&s.min_ret, (unsigned long long)rt);
          }
        }
      }
      if (!leave) m = meta_with(m, ST_RUN, pol);
      r.ctx = ctx; r.kv = kv; r.cpu = cpu; r.pend = pend; r.meta = m;
      c.rs[id] = r;
      accA += dA;
      accP += dP;
      const uint32_t nd = demand_of(ctx, kv, cpu, pend, p.cfg.s_in);
      if (inR) {
        if (leave) { c.R.q[pos].e = INVALID; mark_hole(s, 0, pos); }
        else {                                         // tier 0: running (R16, R14)
          c.R.q[pos].e = id;
          c.R.q[pos].last = (uint32_t)t;
          c.R.dem[pos] = nd;
        }
      } else {
        // a granted waiting entry ends the step running: move it to R
        if (!leave) c.R.put(atomicAdd(&s.n_r, 1u), id, c.W.q[pos].V, (uint32_t)t, nd);
        c.W.q[pos].e = INVALID;
        accW2 += dem;
        mark_hole(s, 1, pos);
      }
    }
    // one shared atomic per warp (64-bit shared atomicAdd is a CAS loop)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      my_tok += __shfl_xor_sync(FULL, my_tok, o);
      my_adm += __shfl_xor_sync(FULL, my_adm, o);
      accA += __shfl_xor_sync(FULL, accA, o);
      accP += __shfl_xor_sync(FULL, accP, o);
      accW2 += __shfl_xor_sync(FULL, accW2, o);
    }
#ifdef AUGSCHED_DEBUG
    // §8(c).4: the step's grants fit the limit (R17: sum g <= B)
    if (lane == 0 && (long long)my_tok > (B > 0 ? B : 0)) err_set(p, 8u);
#endif
    if (lane == 0) {
      if (my_tok) cinc(s, AUGSCHED_R_TOKENS, my_tok);
      if (my_adm) cinc(s, AUGSCHED_R_ADMITTED, my_adm);
      if (accA) warp_add64((unsigned long long*)&s.A, (unsigned long long)accA);
      if (accP) warp_add64((unsigned long long*)&s.P, (unsigned long long)accP);
      if (accW2) warp_add64(&s.w2, 0ull - accW2);
    }
  }
  PT(6);
  phase_bar<3>(nb);
  PT(7);
  compact_list(s, c.R, 0, s.n_r);  // syncs
  compact_list(s, c.W, 1, s.n_w);
  if (tid == 0) {
    if (s.A < 0 || s.P < 0 || s.A + s.P > cap) s.cnt[AUGSCHED_R_ERR] |= 1;
#ifdef AUGSCHED_DEBUG
    // §8(c).4: ledger inside the capacity; a dynamic limit inside its clamp
    if (s.A < 0 || s.P < 0 || s.A + s.P > cap) err_set(p, 8u);
    if (s.ip.budget_mode == AUGSCHED_BUDGET_DYNAMIC) {
      const long long lo = (long long)floor(p.cfg.beta_low * (double)s.ip.target_max);
      const long long hi = (long long)floor(p.cfg.beta_high * (double)s.ip.target_max);
      if (B < lo || B > hi) err_set(p, 8u);
    }
#endif
    s.t = t + 1;                                       // S12
    prep_step(p, s, n);
  }
  PT(8);
#ifdef AUGSCHED_SIM_STATS
  if (tid == 0) s.full = 1;
#endif
  ISYNC();
  return true;
}

// Save the instance's resumable state and publish its record.
__device__ void inst_end(const SimParams& p, SimShm& s) {
  const int tid = ITID;
  const uint32_t inst = s.inst;
  InstHdr& H = p.hdr[inst];
  augsched_result& acc = p.acc[inst];
  ISYNC();
  for (int f = tid; f < AUGSCHED_R_NFIELD; f += SIM_NT) {
    if (f == AUGSCHED_R_MAKESPAN) { if (s.c32[f] > s.cnt[f]) s.cnt[f] = s.c32[f]; }
    else s.cnt[f] += s.c32[f];
  }
  ISYNC();
  if (tid == 0) {
    H.t = s.t; H.A = s.A; H.P = s.P; H.min_ret = s.min_ret; H.next_arr = s.next_arr;
    H.n_r = s.n_r; H.n_w = s.n_w; H.n_pz = s.n_pz; H.n_fin = s.n_fin; H.w2 = s.w2;
    s.cnt[AUGSCHED_R_FINAL_T] = s.t;
    s.cnt[AUGSCHED_R_INCOMPLETE] = s.n - s.n_fin;   // R28
  }
  ISYNC();
  augsched_result& out = p.out[inst];
  for (int f = tid; f < AUGSCHED_R_NFIELD; f += SIM_NT) { acc.f[f] = s.cnt[f]; out.f[f] = s.cnt[f]; }
  for (int b = tid; b < AUGSCHED_NBIN; b += SIM_NT) {
    out.hist_ttft[b] = __ldcg(&acc.hist_ttft[b]);   // written by L2 atomics above
    out.hist_norm[b] = __ldcg(&acc.hist_norm[b]);
  }
}

// Persistent kernel: SIM_WPC one-warp instances per CTA, work stealing over
// instances.  The CTA's instances advance one iteration per CTA barrier.
__global__ void __launch_bounds__(SIM_NT * SIM_WPC, (SIM_MINB / SIM_WPC > 0 ? SIM_MINB / SIM_WPC : 1))
    sim_kernel(const __grid_constant__ SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SimShm& s = reinterpret_cast<SimShm*>(smem_raw)[threadIdx.x / SIM_NT];
  bool active = false, exhausted = false;
#ifdef AUGSCHED_SIM_STATS
  if (ITID == 0) s.full = 0;
#endif
  for (;;) {
    while (!active && !exhausted) {
      if (ITID == 0) s.inst = atomicAdd(p.work, 1u);
      ISYNC();
      const uint32_t inst = s.inst;
      ISYNC();
      if (inst >= p.n_inst) exhausted = true;
      else active = inst_begin(p, s, inst);
    }
    if (SIM_WPC > 1) {
      if (!__syncthreads_or(active)) return;
#ifdef AUGSCHED_SIM_STATS
      // per CTA iteration: the phase times of the slowest full step and the
      // sums over the CTA's full steps
      if (threadIdx.x == 0) {
        SimShm* a = reinterpret_cast<SimShm*>(smem_raw);
        long long best = -1, d[6], bd[6] = {0, 0, 0, 0, 0, 0}, sd[6] = {0, 0, 0, 0, 0, 0};
        int nf = 0;
        for (int w = 0; w < SIM_WPC; ++w) {
          if (!a[w].full) continue;
          a[w].full = 0;
          const long long* q = a[w].pt;
          d[0] = q[1] - q[0]; d[1] = q[2] - q[1]; d[2] = q[3] - q[2]; d[3] = q[4] - q[3];
          d[4] = q[6] - q[5]; d[5] = q[8] - q[7];
          long long tot = 0;
          for (int i = 0; i < 6; ++i) { tot += d[i]; sd[i] += d[i]; }
          if (tot > best) { best = tot; for (int i = 0; i < 6; ++i) bd[i] = d[i]; }
          ++nf;
        }
        if (nf) {
          for (int i = 0; i < 6; ++i) {
            atomicAdd(&g_sim_stats[32 + i], (unsigned long long)bd[i]);
            atomicAdd(&g_sim_stats[40 + i], (unsigned long long)sd[i]);
          }
          atomicAdd(&g_sim_stats[46], (unsigned long long)nf);
          atomicAdd(&g_sim_stats[47], 1ull);
        }
      }
      __syncthreads();
#endif
    } else if (!active) {
      return;
    }
    if (!active) {
      int nb = 0;
      phase_rest(nb);
    } else if (!inst_step(p, s)) {
      inst_end(p, s);
      ISYNC();
      active = false;
    }
  }
}

}  // namespace

size_t sim_smem_bytes() { return SIM_WPC * ((sizeof(SimShm) + 15) & ~size_t(15)); }

#ifdef AUGSCHED_SIM_STATS
extern "C" AUGSCHED_API int augsched_sim_stats(unsigned long long* host, int reset) {
  if (cudaMemcpyFromSymbol(host, g_sim_stats, sizeof(g_sim_stats)) != cudaSuccess) return -3;
  if (reset) {
    static const unsigned long long zero[64] = {};
    if (cudaMemcpyToSymbol(g_sim_stats, zero, sizeof(zero)) != cudaSuccess) return -3;
  }
  return 0;
}
#endif

const void* sim_kernel_ptr() { return reinterpret_cast<const void*>(&sim_kernel); }

cudaError_t launch_sim(const SimParams& p, int grid, size_t smem, cudaStream_t st) {
  sim_kernel<<<grid, SIM_NT * SIM_WPC, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace augsched
