// augsched_simulate: persistent per-instance simulation kernel for sm_100a.
// See sim.cuh for the design; the per-step sequence follows DESIGN.md §"Step
// sequence" (S1..S12), i.e. Algorithm 1 plus the engine model.
#include <cuda_runtime.h>
#include "sim.cuh"
#include "select.cuh"

namespace augsched {

struct __align__(16) SimShm {
  union {
    SelBinsT<SIM_RB> b;              // radix-select histograms (fallback path)
    CandShmT<SIM_CAND> c;            // small candidate lists (fast path)
  } u;
  SelRes res;
  unsigned long long tw[3];          // per-tier demand (clamped to B) of the step
  unsigned int tc[3];                // per-tier queue counts of the step
  unsigned long long rk[2][SIM_NW];  // waiting-tier pop rounds: per-warp smallest key
  unsigned int rw[2][SIM_NW];        //   and its demand (double-buffered by round parity)
  int due;                           // intake or idle handling needed this iteration
  unsigned long long cnt[AUGSCHED_R_NFIELD];
  unsigned int holes[HOLE_CAP];
  unsigned int wtot[SIM_NW + 1];
  Coef coef;                         // per-instance constants (§8(c).1)
  augsched_instance_params ip;
  // instance scalars
  unsigned long long t, tT, min_ret, next_tick;
  long long A, P, A_snap, B, need, freev;
  unsigned long long freed;
  unsigned int next_arr, n_act, n_pz, n_fin, n_holes, n_pholes, wpos;
  unsigned int inst, n_req, r0;
  int run, idle;
};

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t INVALID = 0xffffffffu;

__device__ __forceinline__ void err_set(const SimParams& p, uint32_t bits) { atomicOr(p.err, bits); }

// Block-wide exclusive scan of a 0/1 flag; returns this thread's prefix and
// (in s.wtot[SIM_NW]) the block total.  Contains two __syncthreads.
__device__ __forceinline__ uint32_t block_flag_scan(SimShm& s, bool f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(FULL, f);
  if (lane == 0) s.wtot[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < SIM_NW; ++w) { uint32_t x = s.wtot[w]; s.wtot[w] = acc; acc += x; }
    s.wtot[SIM_NW] = acc;
  }
  __syncthreads();
  return s.wtot[warp] + __popc(b & ((1u << lane) - 1));
}

// Weighted MSD radix select.  Among items i < n for which get(i, key, w)
// returns true (w >= 1, keys unique, key < 2^nbits) find the smallest key k*
// with sum_{key <= k*} w >= D.  Results: s.sel.found (1 found / 0 not: then
// s.sel.total holds the full weight), s.sel.k, s.sel.wbelow = sum_{key < k*} w.
// Weights are clamped to D (exact: every item before k* has w < D).
struct Ctx {
  const SimParams& p;
  SimShm& s;
  const Coef& k;                        // in shared memory (keeps registers free)
  const augsched_instance_params& ip;   // in shared memory
  // arena slices of this instance
  ReqState* rs;
  uint32_t *ac_id, *ac_last, *ac_dem, *pz_id;
  uint64_t* ret;
  double* ac_V;
  uint32_t r0, n, trace;
};

__device__ __forceinline__ uint32_t gen_total(const DevTrace& tr, uint32_t rid) {
  const uint32_t s0 = tr.seg_off[rid], ns = tr.n_seg[rid];
  uint32_t g = 0;
  for (uint32_t q = 0; q < ns; ++q) g += tr.gen_true[s0 + q];
  return g;
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
  atomicAdd(&s.cnt[AUGSCHED_R_RETURNS], 1ull);
  const uint32_t pos = atomicAdd(&s.n_act, 1u);
  c.ac_id[pos] = id | (tier << 30);
  c.ac_V[pos] = V;
  c.ac_last[pos] = r.lastc;  // not reset on return (R14)
  c.ac_dem[pos] = demand_of(ctx, kv, cpu, (int32_t)R, c.p.cfg.s_in);
}


// S3: arrival of request `id` at active position `pos` (Algorithm 1 lines 2-9).
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
  if (ns == 0 || ns > 255) { err_set(c.p, 4u); c.s.cnt[AUGSCHED_R_ERR] |= 4; }  // meta holds 8 bits
  ReqState r;
  r.ctx = 0; r.kv = 0; r.cpu = 0; r.pend = (int32_t)L;
  r.meta = make_meta(0, ST_WAIT, POL_D, ns);
  r.ft = 0; r.lastc = 0;
  r.left = tr.gen_true[s0];
  c.rs[id] = r;
  c.ac_id[pos] = id | (2u << 30);
  c.ac_V[pos] = V;
  c.ac_last[pos] = (uint32_t)t;           // R14, R31
  c.ac_dem[pos] = (uint32_t)L;
}

// Remove the active entries whose ac_id was set to INVALID.
__device__ void compact_active(Ctx& c) {
  SimShm& s = c.s;
  const int tid = threadIdx.x;
  __syncthreads();
  if (s.n_holes == 0) return;
  if (s.n_holes <= HOLE_CAP) {
    if (tid == 0) {
      const uint32_t L = s.n_holes, n = s.n_act, n_new = n - L;
      uint32_t* h = s.holes;
      for (uint32_t a = 1; a < L; ++a) {  // insertion sort (L small)
        uint32_t x = h[a];
        int b = (int)a - 1;
        while (b >= 0 && h[b] > x) { h[b + 1] = h[b]; --b; }
        h[b + 1] = x;
      }
      int j = (int)L - 1;
      int src = (int)n - 1;
      for (uint32_t a = 0; a < L; ++a) {
        const uint32_t hp = h[a];
        if (hp >= n_new) break;
        while (j >= 0 && (int)h[j] == src) { --j; --src; }
        c.ac_id[hp] = c.ac_id[src];
        c.ac_V[hp] = c.ac_V[src];
        c.ac_last[hp] = c.ac_last[src];
        c.ac_dem[hp] = c.ac_dem[src];
        --src;
      }
      s.n_act = n_new;
    }
    __syncthreads();
    return;
  }
  // many removals: in-place tiled stream compaction
  if (tid == 0) s.wpos = 0;
  const uint32_t n = s.n_act;
  for (uint32_t base = 0; base < n; base += SIM_NT) {
    const uint32_t i = base + tid;
    uint32_t id = INVALID, last = 0, dem = 0;
    double V = 0;
    if (i < n) { id = c.ac_id[i]; if (id != INVALID) { V = c.ac_V[i]; last = c.ac_last[i]; dem = c.ac_dem[i]; } }
    const bool keep = id != INVALID;
    const uint32_t pre = block_flag_scan(s, keep);  // syncs: all reads of the tile are done
    const uint32_t w = s.wpos + pre;
    if (keep) { c.ac_id[w] = id; c.ac_V[w] = V; c.ac_last[w] = last; c.ac_dem[w] = dem; }
    __syncthreads();
    if (tid == 0) s.wpos += s.wtot[SIM_NW];
    __syncthreads();
  }
  if (tid == 0) s.n_act = s.wpos;
  __syncthreads();
}

// Remove paused entries marked INVALID (small list; tiled compaction).
__device__ void compact_paused(Ctx& c) {
  SimShm& s = c.s;
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid == 0) s.wpos = 0;
  const uint32_t n = s.n_pz;
  for (uint32_t base = 0; base < n; base += SIM_NT) {
    const uint32_t i = base + tid;
    const uint32_t id = i < n ? c.pz_id[i] : INVALID;
    const bool keep = id != INVALID;
    const uint32_t pre = block_flag_scan(s, keep);
    if (keep) c.pz_id[s.wpos + pre] = id;
    __syncthreads();
    if (tid == 0) s.wpos += s.wtot[SIM_NW];
    __syncthreads();
  }
  if (tid == 0) s.n_pz = s.wpos;
  __syncthreads();
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

__device__ void run_instance(const SimParams& p, SimShm& s, uint64_t* Ksm, uint32_t* Wsm,
                             uint32_t inst) {
  const int tid = threadIdx.x;
  const size_t off = (size_t)inst * p.max_active;
  const Arena& a = p.ar;
  if (tid == 0) { s.coef = make_coef(p.cfg, p.ip[inst]); s.ip = p.ip[inst]; }
  __syncthreads();
  Ctx c{p, s, s.coef, s.ip, a.rs + off, a.ac_id + off, a.ac_last + off, a.ac_dem + off, a.pz_id + off,
        a.ret + off, a.ac_V + off, 0, 0, 0};
  c.trace = p.inst_trace[inst];
  c.r0 = p.tr.req_off[c.trace];
  c.n = p.tr.req_off[c.trace + 1] - c.r0;
  const uint64_t T = p.cfg.t_fwd_ticks;
  const uint32_t n = c.n;
  InstHdr& H = p.hdr[inst];
  augsched_result& acc = p.acc[inst];
  if (n > p.max_active) {  // trace longer than the arena
    if (tid == 0) { err_set(p, 2u); acc.f[AUGSCHED_R_ERR] |= 2; }
    __syncthreads();
    if (tid == 0) p.out[inst] = acc;
    return;
  }
  // ---- load (or initialise) the resumable state -------------------------
  if (tid == 0) {
    if (!H.started) {
      H.t = 0; H.A = 0; H.P = 0; H.min_ret = ~0ull; H.next_arr = 0; H.n_act = 0; H.n_pz = 0;
      H.n_fin = 0; H.started = 1;
    }
    s.t = H.t; s.A = H.A; s.P = H.P; s.min_ret = H.min_ret; s.next_arr = H.next_arr;
    s.n_act = H.n_act; s.n_pz = H.n_pz; s.n_fin = H.n_fin;
    s.next_tick = s.next_arr < n ? p.tr.arr_tick[c.r0 + s.next_arr] : ~0ull;
  }
  for (int f = tid; f < AUGSCHED_R_NFIELD; f += SIM_NT) s.cnt[f] = acc.f[f];
  __syncthreads();
  if (tid == 0) s.cnt[AUGSCHED_R_NREQ] = n;
  const int64_t cap = p.cap;

  // thread 0 prepares iteration s.t: stop rule, S1 snapshot, whether intake
  // or the idle jump must run, and (when no intake is due) the token limit.
  auto prep = [&]() {
    s.run = (s.n_fin < n) && (s.t < p.max_iters);
    s.tT = s.t * T;
    s.A_snap = s.A;
    s.n_holes = 0;
    s.due = s.n_act == 0 || s.tT >= s.min_ret || s.tT >= s.next_tick;
    if (!s.due) s.B = token_limit(p.cfg, c.k, c.ip, cap, s.A, s.P);
    s.tw[0] = s.tw[1] = s.tw[2] = 0;
    s.tc[0] = s.tc[1] = s.tc[2] = 0;
  };
  if (tid == 0) prep();
  __syncthreads();

  for (;;) {
    if (!s.run) break;
    const uint64_t t = s.t, tT = s.tT;
    if (s.due) {
      // ---- S2 returns --------------------------------------------------------
      if (tT >= s.min_ret) {
        const uint32_t npz = s.n_pz;
        for (uint32_t i = tid; i < npz; i += SIM_NT) {
          const uint32_t id = c.pz_id[i];
          if (c.ret[id] <= tT) { do_return(c, id); c.pz_id[i] = INVALID; }
        }
        compact_paused(c);
        if (tid == 0) s.min_ret = ~0ull;
        __syncthreads();
        for (uint32_t i = tid; i < s.n_pz; i += SIM_NT) atomicMin(&s.min_ret, (unsigned long long)c.ret[c.pz_id[i]]);
        __syncthreads();
      }
      // ---- S3 arrivals (ticks are sorted: the arrivals are a prefix) ----------
      if (tT >= s.next_tick) for (;;) {
        const uint32_t j = s.next_arr + tid;
        const bool arrive = j < n && p.tr.arr_tick[c.r0 + j] <= tT;
        const int cnt = __syncthreads_count(arrive);
        if (arrive) do_arrival(c, j, s.n_act + tid, t);
        __syncthreads();
        if (tid == 0) {
          s.n_act += cnt; s.next_arr += cnt; s.cnt[AUGSCHED_R_ARRIVED] += cnt;
          if (cnt < SIM_NT) s.next_tick = s.next_arr < n ? p.tr.arr_tick[c.r0 + s.next_arr] : ~0ull;
        }
        __syncthreads();
        if (cnt < SIM_NT) break;
      }
      // ---- idle jump (not counted) or S4 token limit ---------------------------
      if (tid == 0) {
        s.idle = 0;
        if (s.n_act == 0) {
          uint64_t te = ~0ull;
          if (s.next_arr < n) te = (p.tr.arr_tick[c.r0 + s.next_arr] + T - 1) / T;
          if (s.n_pz > 0) { const uint64_t tr_ = (s.min_ret + T - 1) / T; te = tr_ < te ? tr_ : te; }
          if (te == ~0ull) { s.idle = 2; s.run = 0; }
          else { s.t = te; s.idle = 1; prep(); }
        } else {
          s.B = token_limit(p.cfg, c.k, c.ip, cap, s.A, s.P);
        }
      }
      __syncthreads();
      if (s.idle) continue;
    }
    // ---- S5 keys, per-tier demand, running/swapped candidate lists -----------
    const uint32_t na = s.n_act;
    const long long B = s.B;
    const uint32_t Bc = B > 0 ? (uint32_t)B : 0u;
    const bool in_smem = na <= p.scap;
    uint64_t* K = in_smem ? Ksm : a.kscr + off;
    uint32_t* W = in_smem ? Wsm : a.wscr + off;
    const bool fcfs = c.ip.ranking == AUGSCHED_RANK_FCFS;
    // This thread's two smallest waiting-tier keys (and demands): the first
    // candidates of the pop rounds below.
    uint64_t c1 = ~0ull, c2 = ~0ull;
    uint32_t cw1 = 0, cw2 = 0;
    {
      unsigned long long tw0 = 0, tw1 = 0, tw2 = 0;
      constexpr int U = SIM_UNROLL;  // entries in flight per thread (independent L2 loads)
      const int lane = tid & 31;
      const unsigned lt = (1u << lane) - 1;
      // warp-uniform trip count (the candidate lists use warp ballots)
      for (uint32_t b0 = 0; b0 < na; b0 += SIM_NT * U) {
        uint32_t e[U], l[U], d[U];
        double V[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = b0 + u * SIM_NT + tid;
          if (i < na) { e[u] = c.ac_id[i]; V[u] = c.ac_V[i]; l[u] = c.ac_last[i]; d[u] = c.ac_dem[i]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = b0 + u * SIM_NT + tid;
          uint32_t tier = 3;
          uint64_t Ki = 0;
          if (i < na) {
            tier = e[u] >> 30;
            const uint32_t key = fcfs ? 0u : sched_key(c.k, V[u], t, l[u]);
            Ki = ((uint64_t)tier << 48) | ((uint64_t)key << 16) | (e[u] & 0xFFFF);
            K[i] = Ki;
            W[i] = d[u];
            const uint32_t dc = d[u] < Bc ? d[u] : Bc;
            if (tier == 2) {
              tw2 += dc;
              if (Ki < c2) {
                if (Ki < c1) { c2 = c1; cw2 = cw1; c1 = Ki; cw1 = d[u]; }
                else { c2 = Ki; cw2 = d[u]; }
              }
            } else if (tier == 0) tw0 += dc;
            else tw1 += dc;
          }
          // running / swapped candidate lists, one shared atomic per warp and tier
#pragma unroll
          for (uint32_t tt = 0; tt < 2; ++tt) {
            const unsigned m = __ballot_sync(FULL, tier == tt);
            if (m) {
              const int leader = __ffs(m) - 1;
              uint32_t q0 = 0;
              if (lane == leader) q0 = atomicAdd(&s.tc[tt], (unsigned)__popc(m));
              q0 = __shfl_sync(FULL, q0, leader);
              const uint32_t q = q0 + __popc(m & lt);
              if (tier == tt && q < SIM_CAND) { s.u.c.ck[tt][q] = Ki; s.u.c.cw[tt][q] = d[u]; }
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tw0 += __shfl_xor_sync(FULL, tw0, o);
        tw1 += __shfl_xor_sync(FULL, tw1, o);
        tw2 += __shfl_xor_sync(FULL, tw2, o);
      }
      if ((tid & 31) == 0) {
        if (tw0) atomicAdd(&s.tw[0], tw0);
        if (tw1) atomicAdd(&s.tw[1], tw1);
        if (tw2) atomicAdd(&s.tw[2], tw2);
      }
      if (tid == 0) {
        s.cnt[AUGSCHED_R_BUSY_STEPS] += 1;
        s.cnt[AUGSCHED_R_DECISIONS] += na;
        if (na > s.cnt[AUGSCHED_R_MAXQ]) s.cnt[AUGSCHED_R_MAXQ] = na;
      }
    }
    __syncthreads();
    // ---- S6/S7 order + admission: find the last admitted entry k* --------------
    // Tiers are ordered running < swapped < waiting, so the crossing tier follows
    // from the per-tier totals; within it the crossing comes from a rank select
    // over the (small) candidate list, or from argmin rounds over the waiting
    // tier; the radix select over the whole queue is the fallback.
    {
      const unsigned long long w0 = s.tw[0], w1 = s.tw[1], w2 = s.tw[2];
      const unsigned long long Bu = (unsigned long long)Bc;
      bool done = false;
      if (B <= 0) {
        if (tid == 0) { s.res.found = 1; s.res.k = 0; s.res.wbelow = 0; }  // nothing admitted
        done = true;
      } else if (w0 + w1 + w2 < Bu) {
        if (tid == 0) { s.res.found = 0; s.res.total = w0 + w1 + w2; }    // everything admitted
        done = true;
      } else if (w0 >= Bu) {
        if (s.tc[0] <= SIM_CAND) { select_cand(s, 0, (int)s.tc[0], Bu, 0); done = true; }
      } else if (w0 + w1 >= Bu) {
        if (s.tc[1] <= SIM_CAND) { select_cand(s, 1, (int)s.tc[1], Bu, w0); done = true; }
      } else {
        // waiting tier: pop the smallest remaining waiting keys in order, one
        // per round (one barrier each).  Every thread offers its smallest
        // unconsumed waiting key (c1, then c2, then a rescan of its own
        // entries); the block minimum is the next entry of the order.
        const int lane = tid & 31, warp = tid >> 5;
        unsigned long long wb = w0 + w1;
        uint64_t myk = c1;
        uint32_t myw = cw1;
        int cons = 0;
        for (int r = 0; r < 32; ++r) {
          uint64_t mk = myk;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(FULL, mk, o);
            mk = y < mk ? y : mk;
          }
          const unsigned own = __ballot_sync(FULL, myk == mk);
          if (lane == __ffs(own) - 1) { s.rk[r & 1][warp] = mk; s.rw[r & 1][warp] = myw; }
          __syncthreads();
          uint64_t bk = s.rk[r & 1][0];
          uint32_t bw = s.rw[r & 1][0];
#pragma unroll
          for (int w = 1; w < SIM_NW; ++w) {
            const uint64_t x = s.rk[r & 1][w];
            if (x < bk) { bk = x; bw = s.rw[r & 1][w]; }
          }
          if (bk == ~0ull) break;  // not reachable: w0 + w1 + w2 >= B
          if (wb + bw >= Bu) {
            if (tid == 0) { s.res.found = 1; s.res.k = bk; s.res.wbelow = wb; }
            done = true;
            break;
          }
          wb += bw;
          if (myk == bk) {
            if (++cons == 1) { myk = c2; myw = cw2; }
            else {
              uint64_t nk = ~0ull;
              uint32_t nw = 0;
              for (uint32_t i = tid; i < na; i += SIM_NT) {
                const uint64_t Ki = K[i];
                if ((Ki >> 48) == 2 && Ki > bk && Ki < nk) { nk = Ki; nw = W[i]; }
              }
              myk = nk; myw = nw;
            }
          }
        }
      }
      if (!done) select_arr(s, K, W, na, Bu, KBITS, false);
      __syncthreads();
    }
    const bool found = s.res.found != 0;
    const uint64_t kstar = B > 0 ? s.res.k : 0;
    const uint64_t wb = s.res.wbelow;
    auto grant = [&](uint64_t Ki, uint32_t dem) -> uint32_t {
      if (Ki & KEVICT) return 0u;
      if (B <= 0) return 0u;
      if (!found || Ki < kstar) return dem;
      if (Ki == kstar) return (uint32_t)((uint64_t)B - wb);
      return 0u;
    };
    const long long need = B <= 0 ? 0 : (found ? B : (long long)s.res.total);
    long long freev = cap - s.A - s.P;
    // ---- S8 memory resolution (R20) -------------------------------------------
    if (need > freev) {
      // (1) demote Preserve-paused contexts, kv desc, id asc
      const uint64_t D0 = (uint64_t)(need - freev);
      const uint32_t npz = s.n_pz;
      auto getp = [&](uint32_t i, uint64_t& key, uint32_t& w) {
        const uint32_t id = c.pz_id[i];
        const int32_t kv = c.rs[id].kv;
        if (meta_pol(c.rs[id].meta) != POL_P || kv <= 0) return false;
        key = ((uint64_t)(0xFFFFFFFFu - (uint32_t)kv) << 16) | id;
        w = (uint32_t)kv;
        return true;
      };
      if (tid == 0) { s.tc[0] = 0; s.freed = 0; }
      __syncthreads();
      for (uint32_t i = tid; i < npz; i += SIM_NT) {
        uint64_t key; uint32_t w;
        if (getp(i, key, w)) {
          const uint32_t q = atomicAdd(&s.tc[0], 1u);
          if (q < SIM_CAND) { s.u.c.ck[0][q] = key; s.u.c.cw[0][q] = w; }
        }
      }
      __syncthreads();
      if (s.tc[0] <= SIM_CAND) select_cand(s, 0, (int)s.tc[0], D0, 0);
      else {
        // many Preserve-paused contexts: materialise (key, kv) and select over the arrays
        uint64_t* K2 = a.kscr2 + off;
        uint32_t* W2 = a.wscr2 + off;
        for (uint32_t i = tid; i < npz; i += SIM_NT) {
          uint64_t key = 0; uint32_t w = 0;
          if (!getp(i, key, w)) w = 0;
          K2[i] = key; W2[i] = w;
        }
        __syncthreads();
        select_arr(s, K2, W2, npz, D0, 48, false);
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
            atomicAdd(&s.cnt[AUGSCHED_R_DEMOTIONS], 1ull);
          }
        }
      }
      __syncthreads();
      freev += (long long)s.freed;
      if (tid == 0) { s.P -= (long long)s.freed; s.tc[1] = 0; }
      __syncthreads();
      // (2) evict from the tail of the order over entries with kv + g > 0
      if (need > freev) {
        const uint64_t D1 = (uint64_t)(need - freev);
        for (uint32_t i = tid; i < na; i += SIM_NT) {
          const uint32_t id = c.ac_id[i] & 0xFFFF;
          const uint32_t w = (uint32_t)c.rs[id].kv + grant(K[i], c.ac_dem[i]);
          W[i] = w;
          if (w > 0) {
            const uint32_t q = atomicAdd(&s.tc[1], 1u);
            if (q < SIM_CAND) { s.u.c.ck[1][q] = KMASK - K[i]; s.u.c.cw[1][q] = w; }
          }
        }
        __syncthreads();
        auto gete = [&](uint32_t i, uint64_t& key, uint32_t& w) {
          w = W[i];
          key = KMASK - K[i];
          return w > 0;
        };
        if (s.tc[1] <= SIM_CAND) select_cand(s, 1, (int)s.tc[1], D1, 0);
        else select_arr(s, K, W, na, D1, KBITS, true);
        const bool f1 = s.res.found != 0;
        const uint64_t k1 = s.res.k;
        for (uint32_t i = tid; i < na; i += SIM_NT) {
          uint64_t key; uint32_t w;
          if (gete(i, key, w) && (!f1 || key <= k1)) {
            const uint32_t e = c.ac_id[i];
            const uint32_t id = e & 0xFFFF;
            ReqState r = c.rs[id];
            atomicAdd((unsigned long long*)&s.A, (unsigned long long)(-(long long)r.kv));
            r.kv = 0;
            r.cpu = 0;
            r.meta = meta_with(r.meta, ST_WAIT, meta_pol(r.meta));
            c.rs[id] = r;
            c.ac_id[i] = id | (2u << 30);
            c.ac_dem[i] = demand_of(r.ctx, 0, 0, r.pend, p.cfg.s_in);
            K[i] |= KEVICT;
            atomicAdd(&s.cnt[AUGSCHED_R_EVICTIONS], 1ull);
          }
        }
        __syncthreads();
      }
    }
    // ---- S9 last = t for granted entries; S10 engine advance -------------------
    {
      uint32_t my_tok = 0, my_adm = 0;
      long long accA = 0, accP = 0;
      for (uint32_t i = tid; i < na; i += SIM_NT) {
        const uint64_t Ki = K[i];
        const uint32_t dem = c.ac_dem[i], e = c.ac_id[i];  // independent loads, issued together
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
              atomicAdd(&s.cnt[AUGSCHED_R_COMPLETED], 1ull);
              if (ok) atomicAdd(&s.cnt[AUGSCHED_R_SLO_OK], 1ull);
              if (ok5) atomicAdd(&s.cnt[AUGSCHED_R_SLO_OK_5X], 1ull);
              atomicMax(&s.cnt[AUGSCHED_R_MAKESPAN], (unsigned long long)fin);
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
              if (np == POL_P) { dP += kv; atomicAdd(&s.cnt[AUGSCHED_R_CALLS_PRESERVE], 1ull); }
              else if (np == POL_S) { cpu = ctx; kv = 0; atomicAdd(&s.cnt[AUGSCHED_R_CALLS_SWAP], 1ull); }
              else { kv = 0; atomicAdd(&s.cnt[AUGSCHED_R_CALLS_DISCARD], 1ull); }
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
        if (leave) {
          c.ac_id[i] = INVALID;
          const uint32_t hslot = atomicAdd(&s.n_holes, 1u);
          if (hslot < HOLE_CAP) s.holes[hslot] = i;
        } else {
          c.ac_id[i] = id;                               // tier 0: running (R16)
          c.ac_last[i] = (uint32_t)t;                    // R14
          c.ac_dem[i] = demand_of(ctx, kv, cpu, pend, p.cfg.s_in);
        }
      }
      // one shared atomic per warp (64-bit shared atomicAdd is a CAS loop)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        my_tok += __shfl_xor_sync(FULL, my_tok, o);
        my_adm += __shfl_xor_sync(FULL, my_adm, o);
        accA += __shfl_xor_sync(FULL, accA, o);
        accP += __shfl_xor_sync(FULL, accP, o);
      }
      if ((tid & 31) == 0) {
        if (my_tok) atomicAdd(&s.cnt[AUGSCHED_R_TOKENS], (unsigned long long)my_tok);
        if (my_adm) atomicAdd(&s.cnt[AUGSCHED_R_ADMITTED], (unsigned long long)my_adm);
        if (accA) atomicAdd((unsigned long long*)&s.A, (unsigned long long)accA);
        if (accP) atomicAdd((unsigned long long*)&s.P, (unsigned long long)accP);
      }
    }
    compact_active(c);  // syncs
    if (tid == 0) {
      if (s.A < 0 || s.P < 0 || s.A + s.P > cap) s.cnt[AUGSCHED_R_ERR] |= 1;
      s.t = t + 1;                                       // S12
      prep();
    }
    __syncthreads();
  }
  // ---- save state and results ------------------------------------------------
  __syncthreads();
  if (tid == 0) {
    H.t = s.t; H.A = s.A; H.P = s.P; H.min_ret = s.min_ret; H.next_arr = s.next_arr;
    H.n_act = s.n_act; H.n_pz = s.n_pz; H.n_fin = s.n_fin;
    s.cnt[AUGSCHED_R_FINAL_T] = s.t;
  }
  __syncthreads();
  augsched_result& out = p.out[inst];
  for (int f = tid; f < AUGSCHED_R_NFIELD; f += SIM_NT) { acc.f[f] = s.cnt[f]; out.f[f] = s.cnt[f]; }
  for (int b = tid; b < AUGSCHED_NBIN; b += SIM_NT) {
    out.hist_ttft[b] = __ldcg(&acc.hist_ttft[b]);   // written by L2 atomics above
    out.hist_norm[b] = __ldcg(&acc.hist_norm[b]);
  }
}

__global__ void __launch_bounds__(SIM_NT, SIM_MINB) sim_kernel(const __grid_constant__ SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SimShm& s = *reinterpret_cast<SimShm*>(smem_raw);
  uint64_t* Ksm = reinterpret_cast<uint64_t*>(smem_raw + ((sizeof(SimShm) + 15) & ~size_t(15)));
  uint32_t* Wsm = reinterpret_cast<uint32_t*>(Ksm + p.scap);
  for (;;) {
    if (threadIdx.x == 0) s.inst = atomicAdd(p.work, 1u);
    __syncthreads();
    const uint32_t inst = s.inst;
    if (inst >= p.n_inst) return;
    run_instance(p, s, Ksm, Wsm, inst);
    __syncthreads();
  }
}

}  // namespace

size_t sim_smem_bytes(uint32_t scap) {
  return ((sizeof(SimShm) + 15) & ~size_t(15)) + (size_t)scap * (sizeof(uint64_t) + sizeof(uint32_t));
}

const void* sim_kernel_ptr() { return reinterpret_cast<const void*>(&sim_kernel); }

cudaError_t launch_sim(const SimParams& p, int grid, size_t smem, cudaStream_t st) {
  sim_kernel<<<grid, SIM_NT, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace augsched
