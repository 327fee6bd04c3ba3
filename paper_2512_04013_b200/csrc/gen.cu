// augsched_generate: the counter-based, table-driven workload generator on the
// device (the host twin is tracegen/tablegen.py, which
// documents the scheme).  Every random number is a pure function of (seed,
// trace, request, field), every continuous distribution is sampled through a
// 4,096-level quantile table, and the only floating point is IEEE-exact
// single operations, so the device and the host produce identical traces.
//
// Two passes of one CTA per trace around a scan over traces:
//   gen_count_kernel   gaps -> arrival ticks (block scan), requests kept
//                      (W2: all n_max; W1/W3: arrivals <= horizon), their
//                      segment total
//   gen_offsets_kernel exclusive scans of both over the traces
//   gen_write_kernel   recomputes the arrivals and writes every request and
//                      segment field at its CSR position
#include <cuda_runtime.h>
#include <cstdint>
#include "augsched.h"
#include "model.cuh"

namespace augsched {
namespace {

constexpr int GNT = 256;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t gen_u(uint64_t kt, uint64_t req, uint32_t field) {
  return mix64(kt ^ ((req << 12) | field));
}
__device__ __forceinline__ uint32_t idx12(uint64_t u) { return (uint32_t)(u >> 52); }
__device__ __forceinline__ uint32_t hi32(uint64_t u) { return (uint32_t)(u >> 32); }

// writable view of the caller's output arrays (augsched_trace holds them const)
struct GenOut {
  uint32_t* req_off;
  uint64_t* arr_tick;
  uint32_t *l_pre, *seg_off, *n_seg, *gen_true, *gen_pred, *dur_true;
  float* dur_pred;
  uint32_t* ret_len;
};

struct GenArgs {
  augsched_gen_tables tb;
  uint32_t seed, n_traces, n_max;
  uint64_t horizon;
  const double* scale;       // [n_traces] 1e6 / rate
  uint32_t* cnt;             // [n_traces] requests kept
  uint32_t* segtot;          // [n_traces] their segments
  uint32_t* req_base;        // [n_traces + 1]
  uint32_t* seg_base;        // [n_traces + 1]
  uint32_t* totals;          // [2] n_req, n_seg_total
  GenOut out;                // device arrays to fill
  uint32_t req_cap, seg_cap;
  uint32_t* err;
};

__device__ __forceinline__ uint32_t n_seg_of(const augsched_gen_tables& tb, uint64_t kt, uint64_t j) {
  const uint32_t h2 = hi32(gen_u(kt, j, 2));
  uint32_t cls = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) cls += h2 >= tb.cls_th[c];
  const uint64_t lo = tb.calls_lo[cls], span = (uint64_t)tb.calls_hi[cls] - lo + 1;
  uint64_t calls = lo + (((uint64_t)hi32(gen_u(kt, j, 3)) * span) >> 32);
  if (hi32(gen_u(kt, j, 4)) < tb.nocall_th) calls = 0;
  return (uint32_t)calls + 1;
}

// Block-wide inclusive scan of u64 over GNT threads; carry = sum of earlier chunks.
__device__ __forceinline__ uint64_t block_scan_u64(uint64_t x, uint64_t* wsum, uint64_t& chunk_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint64_t base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < GNT / 32; ++w) {
    const uint64_t v = wsum[w];
    if (w < warp) base += v;
    tot += v;
  }
  chunk_total = tot;
  __syncthreads();
  return base + inc;
}

// Arrival tick of every request of trace k, in chunks; calls f(j, arr) for
// the kept ones and returns the number kept.
template <class F>
__device__ uint32_t arrivals(const GenArgs& a, uint32_t k, uint64_t kt, uint64_t* wsum, F f) {
  const double scale = a.scale[k];
  uint64_t carry = 0;
  uint32_t kept = 0;
  for (uint32_t j0 = 0; j0 < a.n_max; j0 += GNT) {
    const uint32_t j = j0 + threadIdx.x;
    uint64_t gap = 0;
    if (j < a.n_max) gap = (uint64_t)rint(__dmul_rn(a.tb.gap[idx12(gen_u(kt, j, 0))], scale));
    uint64_t tot;
    const uint64_t arr = carry + block_scan_u64(gap, wsum, tot);
    const bool keep = j < a.n_max && (a.horizon == 0 || arr <= a.horizon);
    if (keep) f(j, arr);
    kept += __syncthreads_count(keep);
    carry += tot;
    if (a.horizon != 0 && carry > a.horizon) break;   // later arrivals are past the horizon
  }
  return kept;
}

__global__ void __launch_bounds__(GNT) gen_count_kernel(GenArgs a) {
  __shared__ uint64_t wsum[GNT / 32];
  __shared__ uint32_t segs;
  const uint32_t k = blockIdx.x;
  const uint64_t kt = mix64(((uint64_t)a.seed << 32) | k);
  if (threadIdx.x == 0) segs = 0;
  __syncthreads();
  uint32_t my = 0;
  const uint32_t kept = arrivals(a, k, kt, wsum, [&](uint32_t j, uint64_t) { my += n_seg_of(a.tb, kt, j); });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(FULL, my, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&segs, my);
  __syncthreads();
  if (threadIdx.x == 0) { a.cnt[k] = kept; a.segtot[k] = segs; }
}

// exclusive scans of the per-trace counts (one block, sequential chunks)
__global__ void __launch_bounds__(1024) gen_offsets_kernel(GenArgs a) {
  __shared__ uint64_t ws[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t c0 = 0, c1 = 0;
  for (uint32_t b = 0; b < a.n_traces; b += 1024) {
    const uint32_t k = b + threadIdx.x;
    const uint64_t x0 = k < a.n_traces ? a.cnt[k] : 0, x1 = k < a.n_traces ? a.segtot[k] : 0;
    uint64_t i0 = x0, i1 = x1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y0 = __shfl_up_sync(FULL, i0, o), y1 = __shfl_up_sync(FULL, i1, o);
      if (lane >= o) { i0 += y0; i1 += y1; }
    }
    if (lane == 31) { ws[0][warp] = i0; ws[1][warp] = i1; }
    __syncthreads();
    uint64_t b0 = 0, b1 = 0, t0 = 0, t1 = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) { b0 += ws[0][w]; b1 += ws[1][w]; }
      t0 += ws[0][w]; t1 += ws[1][w];
    }
    if (k < a.n_traces) { a.req_base[k] = (uint32_t)(c0 + b0 + i0 - x0); a.seg_base[k] = (uint32_t)(c1 + b1 + i1 - x1); }
    c0 += t0; c1 += t1;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.req_base[a.n_traces] = (uint32_t)c0;
    a.seg_base[a.n_traces] = (uint32_t)c1;
    a.totals[0] = (uint32_t)c0;
    a.totals[1] = (uint32_t)c1;
    if (c0 > a.req_cap || c1 > a.seg_cap) atomicOr(a.err, 2u);
  }
}

__global__ void __launch_bounds__(GNT) gen_write_kernel(GenArgs a) {
  __shared__ uint64_t wsum[GNT / 32];
  __shared__ uint32_t sw[GNT / 32];
  __shared__ uint32_t seg_carry;
  const uint32_t k = blockIdx.x;
  const uint64_t kt = mix64(((uint64_t)a.seed << 32) | k);
  const uint32_t rb = a.req_base[k], sb = a.seg_base[k];
  if (a.req_base[a.n_traces] > a.req_cap || a.seg_base[a.n_traces] > a.seg_cap) return;
  if (k == 0 && threadIdx.x == 0) a.out.req_off[0] = 0;
  if (threadIdx.x == 0) { a.out.req_off[k + 1] = a.req_base[k + 1]; seg_carry = 0; }
  __syncthreads();
  const augsched_gen_tables& tb = a.tb;
  // requests in chunks: arrival (recomputed), fields, segment offsets (block scan of n_seg)
  const double sc = a.scale[k];
  uint64_t carry = 0;
  for (uint32_t j0 = 0; j0 < a.n_max; j0 += GNT) {
    const uint32_t j = j0 + threadIdx.x;
    uint64_t gap = 0;
    if (j < a.n_max) gap = (uint64_t)rint(__dmul_rn(tb.gap[idx12(gen_u(kt, j, 0))], sc));
    uint64_t tot;
    const uint64_t arr = carry + block_scan_u64(gap, wsum, tot);
    const bool keep = j < a.n_max && (a.horizon == 0 || arr <= a.horizon);
    const uint32_t ns = keep ? n_seg_of(tb, kt, j) : 0u;
    // exclusive scan of n_seg within the chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    uint32_t base = seg_carry, ctot = 0;
#pragma unroll
    for (int w = 0; w < GNT / 32; ++w) {
      if (w < warp) base += sw[w];
      ctot += sw[w];
    }
    if (keep) {
      const uint32_t r = rb + j;
      const uint32_t s0 = sb + base + inc - ns;
      a.out.arr_tick[r] = arr;
      a.out.l_pre[r] = tb.prompt[idx12(gen_u(kt, j, 1))];
      a.out.n_seg[r] = ns;
      a.out.seg_off[r] = s0;
      const uint32_t h2 = hi32(gen_u(kt, j, 2));
      uint32_t cls = 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) cls += h2 >= tb.cls_th[c];
      for (uint32_t sg = 0; sg < ns; ++sg) {
        const uint32_t fb = 16 + 8 * sg;
        const bool last = sg + 1 == ns;
        const uint32_t gt = tb.gen[idx12(gen_u(kt, j, fb + 0))];
        uint32_t gp = gt;
        if (!tb.oracle_pred) {
          int b = 0;
#pragma unroll
          for (int e = 1; e < 8; ++e) b += gt >= tb.edges[e];
          const bool hit = hi32(gen_u(kt, j, fb + 1)) < tb.acc_th;
          const uint32_t shift = 1u + (uint32_t)(((uint64_t)hi32(gen_u(kt, j, fb + 2)) * 7u) >> 32);
          gp = tb.mids[hit ? b : (b + (int)shift) % 8];
        }
        uint32_t dt = 0, rl = 0;
        float dp = 0.0f;
        if (!last) {
          dt = tb.dur[cls * 4096 + idx12(gen_u(kt, j, fb + 3))];
          rl = tb.ret[cls * 4096 + idx12(gen_u(kt, j, fb + 4))];
          const double d = __ddiv_rn((double)dt, 1e6);
          dp = __double2float_rn(tb.oracle_pred ? d : __dmul_rn(d, tb.noise[idx12(gen_u(kt, j, fb + 5))]));
        }
        const uint32_t q = s0 + sg;
        a.out.gen_true[q] = gt;
        a.out.gen_pred[q] = gp;
        a.out.dur_true[q] = dt;
        a.out.dur_pred[q] = dp;
        a.out.ret_len[q] = rl;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) seg_carry += ctot;
    carry += tot;
    __syncthreads();
    if (a.horizon != 0 && carry > a.horizon) break;
  }
}

}  // namespace

int launch_generate(const augsched_gen_tables& tb, const augsched_gen_spec& sp, const augsched_trace& out,
                    uint32_t req_cap, uint32_t seg_cap, uint32_t* scratch, uint32_t* totals, uint32_t* err,
                    cudaStream_t s) {
  GenArgs a;
  a.tb = tb;
  a.seed = sp.seed; a.n_traces = sp.n_traces; a.n_max = sp.n_max; a.horizon = sp.horizon_ticks;
  a.scale = sp.scale;
  a.cnt = scratch;
  a.segtot = scratch + sp.n_traces;
  a.req_base = scratch + 2 * sp.n_traces;
  a.seg_base = scratch + 3 * sp.n_traces + 1;
  a.totals = totals;
  a.out = GenOut{const_cast<uint32_t*>(out.req_off), const_cast<uint64_t*>(out.arr_tick),
                 const_cast<uint32_t*>(out.l_pre), const_cast<uint32_t*>(out.seg_off),
                 const_cast<uint32_t*>(out.n_seg), const_cast<uint32_t*>(out.gen_true),
                 const_cast<uint32_t*>(out.gen_pred), const_cast<uint32_t*>(out.dur_true),
                 const_cast<float*>(out.dur_pred), const_cast<uint32_t*>(out.ret_len)};
  a.req_cap = req_cap; a.seg_cap = seg_cap;
  a.err = err;
  gen_count_kernel<<<sp.n_traces, GNT, 0, s>>>(a);
  gen_offsets_kernel<<<1, 1024, 0, s>>>(a);
  gen_write_kernel<<<sp.n_traces, GNT, 0, s>>>(a);
  return 3;
}

}  // namespace augsched
