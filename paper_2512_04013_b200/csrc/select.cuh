// Block-wide weighted MSD radix select (shared by the simulate and step paths).
//
// Among items i < n for which get(i, key, w) returns true (w >= 1, keys
// unique, key < 2^nbits), find the smallest key k* with
//     sum_{key <= k*} w >= D.
// This is the last entry of the admitted prefix of Algorithm 1's fill loop
// (P:1221-1229 with the chunked last entry of R17) when keys are the
// (tier, score key, id) order and weights the demands; with keys taken from
// the back of the order and weights kv + grant it is the eviction cut of R20.
//
// RB-bit digits from the top (8 for the 256-thread step kernels, 5 = one bin
// per lane for the one-warp simulate CTAs); demand-weighted shared-memory histograms built
// with warp-aggregated atomics (__match_any_sync + __reduce_add_sync), double
// buffered so each pass costs two barriers; a per-bin witness key ends the
// search as soon as the crossing bucket holds a single item.  Weights are
// clamped to D, which is exact: every item before k* has w < D.
#pragma once
#include <cstdint>

#ifndef AUGSCHED_SIM_WPC
#define AUGSCHED_SIM_WPC 16   // instances per simulate CTA (same default as sim.cuh)
#endif

namespace augsched {

// The selection group is NT threads: the whole CTA, or (NT == 32 in a
// simulate CTA that runs several one-warp instances) one warp.
template <int NT>
__device__ __forceinline__ void sel_sync() {
  if (NT == 32 && AUGSCHED_SIM_WPC > 1) __syncwarp();
  else __syncthreads();
}

template <int RB>
struct SelBinsT {
  static constexpr int NB = 1 << RB;
  unsigned long long wbin[2][NB];
  unsigned int cbin[2][NB];
  unsigned long long wkey[2][NB];
};
using SelBins = SelBinsT<8>;

struct SelRes {
  unsigned long long prefix, mask, wbelow, k, total;
  unsigned int cnt;
  int found, done;
};

// convenience for kernels that only need one select
struct SelShm {
  SelBins b;
  SelRes r;
};

// Results: r.found (0: total weight < D, r.total holds it), r.k = k*,
// r.wbelow = sum of weights with key < k*.  Must be called by all NT threads.
template <int NT, int RB, class Get>
__device__ void wselect(SelBinsT<RB>& sb, SelRes& s, uint32_t n, uint64_t D, int nbits, Get get) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NB = 1 << RB;
  static_assert(NB >= 32 && NB % 32 == 0, "one warp scans the bins in 32-wide chunks");
  const int tid = threadIdx.x % NT, lane = tid & 31, warp = tid >> 5;
  const uint32_t Dc = (uint32_t)(D < (1ull << 26) ? D : (1ull << 26));
  sel_sync<NT>();
  if (tid == 0) {
    s.prefix = 0; s.mask = 0; s.wbelow = 0; s.found = 0; s.done = 0; s.total = 0; s.cnt = 0;
    s.k = 0;
  }
  for (int b = tid; b < NB; b += NT) { sb.wbin[0][b] = 0; sb.cbin[0][b] = 0; }
  sel_sync<NT>();
  int hi = nbits, pb = 0;
  while (hi > 0) {
    const int lo = hi > RB ? hi - RB : 0;
    const uint32_t dmask = (1u << (hi - lo)) - 1;
    const uint64_t prefix = s.prefix, mask = s.mask;
    unsigned long long* wbin = sb.wbin[pb];
    unsigned int* cbin = sb.cbin[pb];
    unsigned long long* wkey = sb.wkey[pb];
    for (int b = tid; b < NB; b += NT) { sb.wbin[pb ^ 1][b] = 0; sb.cbin[pb ^ 1][b] = 0; }
    for (uint32_t base = 0; base < n; base += NT) {
      const uint32_t i = base + tid;
      int dig = -1;
      uint32_t w = 0;
      uint64_t key = 0;
      if (i < n) {
        uint32_t wi;
        if (get(i, key, wi) && (key & mask) == prefix) {
          dig = (int)((key >> lo) & dmask);
          w = wi < Dc ? wi : Dc;
        }
      }
      const unsigned peers = __match_any_sync(FULL, dig);
      if (dig >= 0) {
        const unsigned sum = __reduce_add_sync(peers, w);
        if (lane == __ffs(peers) - 1) {
          atomicAdd(&wbin[dig], (unsigned long long)sum);
          atomicAdd(&cbin[dig], (unsigned)__popc(peers));
          atomicExch(&wkey[dig], (unsigned long long)key);   // a witness: read only when the bin holds one item
        }
      }
    }
    sel_sync<NT>();
    if (warp == 0) {
      unsigned long long run = s.wbelow;
      int bin = -1;
      unsigned long long wb = 0;
#pragma unroll 1
      for (int q = 0; q < NB / 32; ++q) {
        const int b = q * 32 + lane;
        const unsigned long long w = wbin[b];
        unsigned long long inc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long v = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += v;
        }
        const unsigned bal = __ballot_sync(FULL, w > 0 && run + inc >= D);
        if (bal) {
          const int f = __ffs(bal) - 1;
          bin = q * 32 + f;
          wb = run + __shfl_sync(FULL, inc - w, f);
          break;
        }
        run += __shfl_sync(FULL, inc, 31);
      }
      if (lane == 0) {
        if (bin < 0) {
          s.found = 0; s.done = 1; s.total = run;
        } else {
          s.prefix = prefix | ((uint64_t)bin << lo);
          s.mask = mask | ((uint64_t)dmask << lo);
          s.wbelow = wb;
          s.cnt = cbin[bin];
          s.found = 1;
          if (lo == 0) { s.done = 1; s.k = s.prefix; }
          else if (s.cnt == 1) { s.done = 1; s.k = wkey[bin]; }
        }
      }
    }
    sel_sync<NT>();
    if (s.done) break;
    hi = lo;
    pb ^= 1;
  }
}

template <int NT, class Get>
__device__ __forceinline__ void wselect(SelShm& s, uint32_t n, uint64_t D, int nbits, Get get) {
  wselect<NT, 8>(s.b, s.r, n, D, nbits, get);
}

// Small-candidate variant: m <= C (key, weight) pairs in shared memory.
// Each candidate's rank is counted against all others (keys unique), pairs
// are scattered to rank order, and one warp scans the weights for the
// crossing.  Results in r as for wselect, with wbelow offset by w0 (the
// weight of everything ordered before the candidate set).
template <int C>
struct CandShmT {
  static constexpr int CAP = C;
  unsigned long long ck[2][C];
  unsigned int cw[2][C];
  unsigned long long rk[C];
  unsigned int rw[C];
};

template <int NT, int C>
__device__ void rank_select(CandShmT<C>& c, int list, SelRes& r, int m, uint64_t D, uint64_t w0) {
  constexpr unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x % NT, lane = tid & 31;
  const unsigned long long* ck = c.ck[list];
  const unsigned int* cw = c.cw[list];
  for (int a = tid; a < m; a += NT) {
    const unsigned long long key = ck[a];
    int rk = 0;
#pragma unroll 4
    for (int j = 0; j < m; ++j) rk += ck[j] < key;
    c.rk[rk] = key;
    c.rw[rk] = cw[a];
  }
  sel_sync<NT>();
  if (tid < 32) {
    unsigned long long run = w0;
    int hit = -1;
    unsigned long long wb = 0;
    for (int q = 0; q < m; q += 32) {
      const int j = q + lane;
      const unsigned long long w = j < m ? c.rw[j] : 0ull;
      unsigned long long inc = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
      }
      const unsigned bal = __ballot_sync(FULL, j < m && run + inc >= D);
      if (bal) {
        const int f = __ffs(bal) - 1;
        hit = q + f;
        wb = run + __shfl_sync(FULL, inc - w, f);
        break;
      }
      run += __shfl_sync(FULL, inc, 31);
    }
    if (lane == 0) {
      if (hit < 0) { r.found = 0; r.total = run; }
      else { r.found = 1; r.k = c.rk[hit]; r.wbelow = wb; }
    }
  }
  sel_sync<NT>();
}

}  // namespace augsched
