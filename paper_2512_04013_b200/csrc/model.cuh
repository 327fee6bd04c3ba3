// Device-side arithmetic of the AugServe scheduling method (arXiv 2512.04013).
// Every binary64 operation is an explicit round-to-nearest intrinsic so the
// result does not depend on FMA contraction (reading R3 in DESIGN.md); the
// translation unit is additionally compiled with -fmad=false.
#pragma once
#include <cstdint>
#include "augsched.h"

namespace augsched {

enum : int { POL_P = 0, POL_S = 1, POL_D = 2 };
// request status (cold state) and queue tier (active list)
enum : uint32_t { ST_NONE = 0, ST_RUN = 1, ST_SWAP = 2, ST_WAIT = 3, ST_PAUSED = 4, ST_DONE = 5 };

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double u2d(uint64_t x) { return __ull2double_rn(x); }

// Per-instance constants: §8(c).1 "Coefficients", computed once per instance.
struct Coef {
  double M, Ts, N, Sout, alpha;
  double cPre;   // 1/2 M T / N      (Eq.9, Eq.17)
  double cDec;   // M T              (Eq.10, Eq.19)
  double cSout;  // 1/2 M T / S_out  (Eq.12, Eq.23)
  double cSin;   // 1/2 M T / S_in   (Eq.16)
  double cPro;   // M T / N          (Eq.18)
  uint64_t n_fwd;
  int64_t lo, hi;  // clamp bounds of P:749
};

__device__ __forceinline__ Coef make_coef(const augsched_config& c,
                                          const augsched_instance_params& p) {
  Coef k;
  k.M = u2d(c.m_per_token);
  k.Ts = ddiv(u2d(c.t_fwd_ticks), 1e6);
  k.N = u2d(p.target_max);             // N^fwd_max := target_max (R9)
  k.n_fwd = p.target_max;
  k.Sout = u2d(c.s_out);
  k.alpha = p.alpha;
  const double hmt = dmul(dmul(0.5, k.M), k.Ts);
  k.cPre = ddiv(hmt, k.N);
  k.cDec = dmul(k.M, k.Ts);
  k.cSout = ddiv(hmt, k.Sout);
  k.cSin = ddiv(hmt, u2d(c.s_in));
  k.cPro = ddiv(dmul(k.M, k.Ts), k.N);
  k.lo = (int64_t)floor(dmul(c.beta_low, u2d(p.target_max)));
  k.hi = (int64_t)floor(dmul(c.beta_high, u2d(p.target_max)));
  return k;
}

// Eq.4-8: wastes of the three context policies and their argmin; ties
// Preserve > Swap > Discard (R8).  C, Co in tokens; Ti predicted seconds.
__device__ __forceinline__ int select_policy(const Coef& k, uint64_t C, double Ti, uint64_t Co,
                                             uint32_t policy_mode) {
  if (policy_mode == AUGSCHED_POLICY_PRESERVE) return POL_P;
  if (policy_mode == AUGSCHED_POLICY_SWAP) return POL_S;
  if (policy_mode == AUGSCHED_POLICY_DISCARD) return POL_D;
  const double c = u2d(C);
  const double wP = dmul(dmul(Ti, c), k.M);                                  // Eq.4
  const double Trc = dmul(u2d((C + k.n_fwd - 1) / k.n_fwd), k.Ts);           // T^fwd(C), R6
  const double wD = dadd(dmul(dmul(Trc, c), k.M), dmul(dmul(Trc, u2d(Co)), k.M));  // Eq.5
  const double wS = dmul(dmul(dmul(2.0, dmul(ddiv(c, k.Sout), k.Ts)), k.N), k.M);  // Eq.6
  if (wP <= wS && wP <= wD) return POL_P;
  if (wS <= wD) return POL_S;
  return POL_D;
}

// Eq.9-15: Stage I value of policy `pol` (no call -> Discard form, R11).
__device__ __forceinline__ double stage1(const Coef& k, uint64_t Lpre, uint64_t Oh, double A, int pol) {
  const double L = u2d(Lpre), O = u2d(Oh);
  const double pre = dmul(k.cPre, dmul(L, L));
  const double dec = dmul(k.cDec, dadd(dmul(L, O), dmul(0.5, dmul(O, O))));
  const double LO = dadd(L, O);
  if (pol == POL_P) return dadd(dadd(pre, dec), dmul(dmul(k.M, LO), A));
  if (pol == POL_S) return dadd(dadd(pre, dec), dmul(k.cSout, dmul(LO, LO)));
  return dadd(pre, dec);
}

// Eq.16-22: Stage II value under the applied policy.
__device__ __forceinline__ double stage2(const Coef& k, uint64_t Ltot, uint64_t Rr, uint64_t On, int pol) {
  const double Lt = u2d(Ltot), R = u2d(Rr), O = u2d(On);
  const double pro = dmul(k.cPro, dadd(dmul(Lt, R), dmul(0.5, dmul(R, R))));
  const double dp = dmul(k.cDec, dadd(dmul(dadd(Lt, R), O), dmul(0.5, dmul(O, O))));
  if (pol == POL_P) return dadd(pro, dp);
  if (pol == POL_S) return dadd(dadd(dmul(k.cSin, dmul(Lt, Lt)), pro), dp);
  return dadd(dadd(dmul(k.cPre, dmul(Lt, Lt)), pro), dp);
}

// Eq.23-25: final value with the next round's predicted policy.
__device__ __forceinline__ double final_value(const Coef& k, double V2, uint64_t X, int nx, double An) {
  const double x = u2d(X);
  if (nx == POL_S) return dadd(V2, dmul(k.cSout, dmul(x, x)));
  if (nx == POL_P) return dadd(V2, dmul(dmul(k.M, x), An));
  return V2;
}

// Stage I value of an arrival (Algorithm 1 lines 2-9; R4, R5, R7, R11).
__device__ __forceinline__ double intake_stage1(const Coef& k, uint32_t pm, uint64_t L, uint64_t O,
                                                double A, bool has_call, uint64_t A_snap) {
  if (!has_call) return stage1(k, L, O, 0.0, POL_D);
  return stage1(k, L, O, A, select_policy(k, L + O, A, A_snap, pm));
}

// Stage II + final value of a return (Algorithm 1 lines 10-24; R12).
__device__ __forceinline__ double intake_stage2(const Coef& k, uint32_t pm, int pol, uint64_t Lt,
                                                uint64_t R, uint64_t On, double An, bool has_next,
                                                uint64_t A_snap) {
  const double V2 = stage2(k, Lt, R, On, pol);
  if (!has_next) return V2;
  const uint64_t X = Lt + R + On;
  return final_value(k, V2, X, select_policy(k, X, An, A_snap, pm), An);
}

// Eq.26 with R1 (waiting lowers the score) and R3 (one RN to fp32, then the
// order-preserving u32 map).
__device__ __forceinline__ uint32_t sched_key(const Coef& k, double V, uint64_t now, uint64_t last) {
  const double w = dmul(u2d(now - last), k.Ts);
  const double s = dsub(V, dmul(k.alpha, w));
  const uint32_t u = __float_as_uint(__double2float_rn(s));
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Random scheduling (reading B8): SplitMix64 output function and the
// per-iteration key of request `id`.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t random_key(uint32_t seed, uint32_t id, uint64_t t) {
  return (uint32_t)(mix64(mix64(((uint64_t)seed << 32) | id) ^ t) >> 32);
}

// Reading B12: the time-invariant form V + alpha*(last*T) of
// Eq.26's score, one RN to fp32 and the same order-preserving map.
__device__ __forceinline__ uint32_t ti_key(const Coef& k, double V, uint64_t last) {
  const double s = dadd(V, dmul(k.alpha, dmul(u2d(last), k.Ts)));
  const uint32_t u = __float_as_uint(__double2float_rn(s));
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Score key of a queued request under the instance's ranking mode.
__device__ __forceinline__ uint32_t rank_key(const Coef& k, const augsched_instance_params& ip, double V,
                                             uint64_t now, uint64_t last, uint32_t id) {
  if (ip.ranking == AUGSCHED_RANK_FCFS) return 0u;
  if (ip.ranking == AUGSCHED_RANK_RANDOM) return random_key(ip.rank_seed, id, now);
  if (ip.ranking == AUGSCHED_RANK_AUGSERVE_TI) return ti_key(k, V, last);
  return sched_key(k, V, now, last);
}

// Eq.27-32 + clamp in whole tokens (R19); static mode returns l_static.
__device__ __forceinline__ int64_t token_limit(const augsched_config& c, const Coef& k,
                                               const augsched_instance_params& p, int64_t cap,
                                               int64_t A, int64_t P) {
  if (p.budget_mode == AUGSCHED_BUDGET_STATIC) return (int64_t)p.l_static;
  const int64_t fr = cap - A - P;
  int64_t raw = (fr > 0 ? fr : 0) + (int64_t)(((uint64_t)c.gamma_num * (uint64_t)P) / c.gamma_den);
  raw = raw < k.lo ? k.lo : raw;
  return raw > k.hi ? k.hi : raw;
}

// Demand of a queued request (R17, R18): swap-in chunk, else recompute +
// prefill/assimilation, else one decode token.
__device__ __forceinline__ uint32_t demand_of(int32_t ctx, int32_t kv, int32_t cpu, int32_t pend,
                                              uint32_t s_in) {
  if (cpu > 0) return (uint32_t)cpu < s_in ? (uint32_t)cpu : s_in;
  const int32_t todo = (ctx - kv) + pend;
  return todo > 0 ? (uint32_t)todo : 1u;
}

__device__ __forceinline__ uint32_t hist_bin(uint64_t v) {
  if (v < 16) return (uint32_t)v;
  const int e = 63 - __clzll((long long)v);
  const uint64_t b = 16 + (uint64_t)(e - 4) * 4 + ((v >> (e - 2)) & 3);
  return b < AUGSCHED_NBIN ? (uint32_t)b : AUGSCHED_NBIN - 1;
}

}  // namespace augsched
