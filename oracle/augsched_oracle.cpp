// ============================================================================
// augsched ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU transcription of AugServe's scheduler
// (arXiv 2512.04013, /root/reference/PAPER.md, "P:n" = line n) driven by the
// execution model and readings R1-R35 of SURVEY.md §8(c) (also listed in
// DESIGN.md).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no
// code, header, table or constant with the CUDA path in
// paper_2512_04013_b200/; its only common input is the numpy trace produced by
// tracegen/.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (no FMA
// contraction: every double op is one IEEE round-to-nearest operation, R3).
//
// Pins (tests/test_oracle_*.py): SPEC worked examples,
// the hand-worked schedules G3-G8 of SURVEY §8(c).3, brute force over all n! orders / 2^n subsets for
// n <= 7, and the invariants of SURVEY §8(c).4.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <tuple>
#include <vector>

extern "C" {

// ---------------------------------------------------------------- config ---
struct OCfg {                 // system constants (SPEC SimConfig S:29-46)
  uint64_t m_per_token;       // M, bytes of KV per token
  uint64_t g_total, g_model, g_runtime, g_safety;  // Eq.29 G terms
  uint64_t t_fwd_ticks;       // T^fwd in integer microsecond ticks (R24)
  uint32_t s_in, s_out;       // S^fwd_in / S^fwd_out tokens per iteration
  uint32_t gamma_num, gamma_den;  // gamma of Eq.31 as a rational (R19)
  double beta_low, beta_high; // clamp factors
};

struct OInst {                // per-instance sweep parameters
  uint32_t target_max;        // target_max; also N^fwd_max in costs (R9)
  uint32_t l_static;          // static batch token limit (budget_mode 1)
  double alpha;               // anti-starvation coefficient (Eq.26)
  uint64_t slo_ttft_ticks;    // TTFT SLO
  uint32_t slo_norm_num, slo_norm_den;  // normalized latency < num/den * T
  uint32_t ranking;           // 0 AugServe value order, 1 FCFS, 2 random, 3 time-invariant (B12)
  uint32_t budget_mode;       // 0 dynamic (Eq.27-32), 1 static
  uint32_t policy_mode;       // 0 argmin (Eq.7-8), 1 Preserve, 2 Swap, 3 Discard
  uint32_t rank_seed;         // seed of random scheduling (ranking 2)
};

struct OTrace {               // CSR trace set produced by tracegen/
  const uint32_t* req_off;
  const uint64_t* arr_tick;
  const uint32_t* l_pre;
  const uint32_t* seg_off;
  const uint32_t* n_seg;
  const uint32_t* gen_true;
  const uint32_t* gen_pred;
  const uint32_t* dur_true;
  const float* dur_pred;
  const uint32_t* ret_len;
};

enum { O_NFIELD = 24, O_NBIN = 160 };
struct OResult {
  uint64_t f[O_NFIELD];       // see field list in oracle/__init__.py
  uint32_t hist_ttft[O_NBIN];
  uint32_t hist_norm[O_NBIN];
};

}  // extern "C"

namespace {

enum Pol { PRESERVE = 0, SWAP = 1, DISCARD = 2 };
enum Status { NOT_ARRIVED = 0, RUNNING = 1, SWAPPED = 2, WAITING = 3, PAUSED = 4, FINISHED = 5 };

// Coefficients of §8(c).1, computed in double, left to right.
struct Coef {
  double M, Ts, N, Sin, Sout;
  double cPre, cDec, cSout, cSin, cPro;
  uint64_t n_fwd;
};

Coef make_coef(const OCfg& c, uint32_t target_max) {
  Coef k;
  k.M = (double)c.m_per_token;
  k.Ts = (double)c.t_fwd_ticks / 1e6;       // seconds per iteration (reading: division)
  k.N = (double)target_max;                 // N^fwd_max = target_max (R9)
  k.n_fwd = target_max;
  k.Sin = (double)c.s_in;
  k.Sout = (double)c.s_out;
  k.cPre = ((0.5 * k.M) * k.Ts) / k.N;      // Eq.9 / Eq.17: 1/2 M T / N
  k.cDec = k.M * k.Ts;                      // Eq.10 / Eq.19: M T
  k.cSout = ((0.5 * k.M) * k.Ts) / k.Sout;  // Eq.12 / Eq.23: 1/2 M T / S_out
  k.cSin = ((0.5 * k.M) * k.Ts) / k.Sin;    // Eq.16: 1/2 M T / S_in
  k.cPro = (k.M * k.Ts) / k.N;              // Eq.18: M T / N
  return k;
}

// ---- Eq.4-8: memory waste of each policy and the argmin ------
// Eq.4  Waste^P = T^INT * C * M
double waste_preserve(const Coef& k, double Ti, uint64_t C) { return (Ti * (double)C) * k.M; }
// Eq.5  Waste^D = T^fwd(C) C M + T^fwd(C) C_other M, T^fwd(C) = ceil(C/N) T (R6)
double waste_discard(const Coef& k, uint64_t C, uint64_t Co) {
  double Trc = (double)((C + k.n_fwd - 1) / k.n_fwd) * k.Ts;
  return ((Trc * (double)C) * k.M) + ((Trc * (double)Co) * k.M);
}
// Eq.6  Waste^S = 2 T^swap(C) N^fwd_max M, T^swap(C) = (C / S_out) T (R6)
double waste_swap(const Coef& k, uint64_t C) {
  return ((2.0 * (((double)C / k.Sout) * k.Ts)) * k.N) * k.M;
}
// Eq.7-8 argmin; ties Preserve > Swap > Discard (R8).
int select_policy(const Coef& k, uint64_t C, double Ti, uint64_t Co, uint32_t policy_mode) {
  if (policy_mode == 1) return PRESERVE;
  if (policy_mode == 2) return SWAP;
  if (policy_mode == 3) return DISCARD;
  double wP = waste_preserve(k, Ti, C);
  double wD = waste_discard(k, C, Co);
  double wS = waste_swap(k, C);
  if (wP <= wS && wP <= wD) return PRESERVE;
  if (wS <= wD) return SWAP;
  return DISCARD;
}

// ---- Eq.9-15: Stage I value -----------------------------------
double stage1_value(const Coef& k, uint64_t Lpre, uint64_t O, double A, int pol) {
  double L = (double)Lpre, Od = (double)O;
  double pre = k.cPre * (L * L);                       // Eq.9
  double dec = k.cDec * ((L * Od) + 0.5 * (Od * Od));  // Eq.10
  double api = (k.M * (L + Od)) * A;                   // Eq.11
  double so = k.cSout * ((L + Od) * (L + Od));         // Eq.12
  if (pol == PRESERVE) return (pre + dec) + api;       // Eq.13
  if (pol == SWAP) return (pre + dec) + so;            // Eq.15
  return pre + dec;                                    // Eq.14 (also: no call, R11)
}

// ---- Eq.16-22: Stage II value ---------------------------------
double stage2_value(const Coef& k, uint64_t Ltot, uint64_t Rret, uint64_t Onext, int pol) {
  double Lt = (double)Ltot, R = (double)Rret, O = (double)Onext;
  double si = k.cSin * (Lt * Lt);                             // Eq.16
  double rc = k.cPre * (Lt * Lt);                             // Eq.17
  double pro = k.cPro * ((Lt * R) + 0.5 * (R * R));           // Eq.18
  double dp = k.cDec * (((Lt + R) * O) + 0.5 * (O * O));      // Eq.19
  if (pol == PRESERVE) return pro + dp;                       // Eq.20
  if (pol == SWAP) return (si + pro) + dp;                    // Eq.21
  return (rc + pro) + dp;                                     // Eq.22
}

// ---- Eq.23-25: final value ------------------------------------
double final_value(const Coef& k, double V2, uint64_t X, int next_pol, double Anext) {
  double x = (double)X;
  if (next_pol == SWAP) return V2 + k.cSout * (x * x);        // Eq.23
  if (next_pol == PRESERVE) return V2 + (k.M * x) * Anext;    // Eq.24
  return V2;                                                  // Eq.25
}

// ---- Eq.26 with R1 (sign) and R3 (fp32 key) --------------------------------
uint32_t sched_key(double V, double alpha, double Ts, uint64_t now, uint64_t last) {
  double w = (double)(now - last) * Ts;   // waiting time in seconds (R15)
  double s = V - (alpha * w);             // V_sched, ascending = scheduled first (R1)
  float f = (float)s;                     // one RN conversion to fp32 (R3)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving u32
}

// ---- random scheduling ("shuffle the request order") ----------
// Reading B8: a fresh shuffle every iteration, drawn from a
// counter-based generator so both implementations draw the same numbers:
// the SplitMix64 output function applied twice, to (seed << 32 | id) and then
// xor-ed with the iteration; the key is the high 32 bits.
uint64_t splitmix64_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint32_t random_key(uint32_t seed, uint32_t id, uint64_t t) {
  const uint64_t a = splitmix64_mix(((uint64_t)seed << 32) | id);
  return (uint32_t)(splitmix64_mix(a ^ t) >> 32);
}

// Reading B12: the time-invariant form of Eq.26.  Between two
// events V - alpha*(now - last)*T and V + alpha*last*T differ by the same
// alpha*now*T for every request, so they rank alike in exact arithmetic;
// this form is rounded once to fp32 like R3.
uint32_t ti_key(double V, double alpha, double Ts, uint64_t last) {
  double s = V + (alpha * ((double)last * Ts));
  float f = (float)s;
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// The order key of a queued request: Eq.26 value order, FCFS, random or the
// time-invariant value order.
uint32_t order_key(const OInst& ip, double V, double Ts, uint64_t now, uint64_t last, uint32_t id) {
  if (ip.ranking == 1) return 0u;                        // FCFS (R33)
  if (ip.ranking == 2) return random_key(ip.rank_seed, id, now);
  if (ip.ranking == 3) return ti_key(V, ip.alpha, Ts, last);
  return sched_key(V, ip.alpha, Ts, now, last);
}

// ---- Eq.27-32 + clamp (Algorithm 1 lines 25-27) ---------------
struct Bounds { int64_t lo, hi; };
Bounds clamp_bounds(const OCfg& c, uint32_t target_max) {
  Bounds b;
  b.lo = (int64_t)std::floor(c.beta_low * (double)target_max);
  b.hi = (int64_t)std::floor(c.beta_high * (double)target_max);
  return b;
}
int64_t cap_tokens(const OCfg& c) {  // floor((G_total - G_fixed)/M) (Eq.29-32, R19)
  uint64_t fixed = c.g_model + c.g_runtime + c.g_safety;
  return (int64_t)((c.g_total - fixed) / c.m_per_token);
}
int64_t token_budget(const OCfg& c, int64_t cap, int64_t A, int64_t P, Bounds b) {
  int64_t free_ = cap - A - P;                                    // Eq.30 / M
  int64_t raw = std::max<int64_t>(free_, 0) +
                (int64_t)(((uint64_t)c.gamma_num * (uint64_t)P) / c.gamma_den);  // Eq.31-32
  return std::min(std::max(raw, b.lo), b.hi);                     // clamp
}

uint32_t hist_bin(uint64_t v) {  // integer log-linear bins, 4 per octave
  if (v < 16) return (uint32_t)v;
  int e = 63 - __builtin_clzll(v);
  uint64_t b = 16 + (uint64_t)(e - 4) * 4 + ((v >> (e - 2)) & 3);
  return (uint32_t)std::min<uint64_t>(b, O_NBIN - 1);
}

// ---------------------------------------------------------------------------
// One simulated serving instance: Algorithm 1 in the step
// order S1..S12 of SURVEY §8(c).1.
// ---------------------------------------------------------------------------
struct Req {
  int status = NOT_ARRIVED;
  uint32_t seg = 0, gen_done = 0;
  int64_t ctx = 0, kv = 0, cpu = 0, pend = 0;
  double V = 0;
  uint64_t last = 0;
  int pol = DISCARD;          // applied policy S~ of the outstanding call
  uint64_t ret_tick = 0;
  int64_t ft = -1;            // iteration index after which the first token exists
  uint64_t gen_total = 0;
};

enum Field {
  F_NREQ, F_ARRIVED, F_COMPLETED, F_SLO_OK, F_SLO_OK5, F_BUSY, F_DECISIONS, F_EVICT,
  F_DEMOTE, F_CALL_P, F_CALL_S, F_CALL_D, F_RETURNS, F_TOKENS, F_FINAL_T, F_MAKESPAN,
  F_SUM_TTFT, F_SUM_E2E, F_SUM_GEN, F_ADMITTED, F_ERR, F_MAXQ, F_INCOMPLETE, F_R23
};

int64_t demand_of(const Req& r, int64_t s_in) {  // a6 demand (R17, R18)
  if (r.cpu > 0) return std::min(r.cpu, s_in);     // swap-in chunk
  int64_t todo = (r.ctx - r.kv) + r.pend;          // recompute + prefill/assimilation
  if (todo > 0) return todo;
  return 1;                                        // decode
}

void simulate_one(const OCfg& cfg, const OInst& ip, const OTrace& tr, uint32_t trace_id,
                  uint64_t max_iters, OResult* res, int64_t* ft_out = nullptr,
                  int64_t* fin_out = nullptr) {
  std::memset(res, 0, sizeof(OResult));
  const Coef k = make_coef(cfg, ip.target_max);
  const Bounds bnd = clamp_bounds(cfg, ip.target_max);
  const int64_t cap = cap_tokens(cfg);
  const uint64_t T = cfg.t_fwd_ticks;
  const uint32_t r0 = tr.req_off[trace_id], n = tr.req_off[trace_id + 1] - r0;
  std::vector<Req> R(n);
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t s0 = tr.seg_off[r0 + i];
    for (uint32_t s = 0; s < tr.n_seg[r0 + i]; ++s) R[i].gen_total += tr.gen_true[s0 + s];
  }
  auto seg = [&](uint32_t i, uint32_t s) { return tr.seg_off[r0 + i] + s; };
  auto nseg = [&](uint32_t i) { return tr.n_seg[r0 + i]; };

  uint64_t* F = res->f;
  F[F_NREQ] = n;
  int64_t A = 0, P = 0;          // ledger in tokens: active KV, Preserve-paused KV
  uint32_t next_arr = 0, n_fin = 0;
  std::vector<uint32_t> active;  // ids in RUNNING u SWAPPED u WAITING
  std::vector<uint32_t> paused;  // ids in PAUSED
  uint64_t t = 0;
  while (n_fin < n && t < max_iters) {
    // S1 snapshot
    const int64_t A_snap = A;
    // S2 returns, in id order (Algorithm 1 lines 10-24; Eq.16-25)
    std::vector<uint32_t> ret_ids;
    for (uint32_t id : paused)
      if (R[id].ret_tick <= t * T) ret_ids.push_back(id);
    std::sort(ret_ids.begin(), ret_ids.end());
    for (uint32_t id : ret_ids) {
      Req& r = R[id];
      uint32_t kk = r.seg;                       // call k follows segment k
      uint64_t Lt = (uint64_t)r.ctx;             // L^total before the call
      uint64_t Rr = tr.ret_len[seg(id, kk)];     // actual return length
      uint64_t On = tr.gen_pred[seg(id, kk + 1)];
      double V2 = stage2_value(k, Lt, Rr, On, r.pol);
      bool has_next = kk + 1 < nseg(id) - 1;
      if (has_next) {
        double An = (double)tr.dur_pred[seg(id, kk + 1)];
        uint64_t X = Lt + Rr + On;
        int nx = select_policy(k, X, An, (uint64_t)A_snap, ip.policy_mode);  // R12
        r.V = final_value(k, V2, X, nx, An);
      } else {
        r.V = V2;                                // no next call (R11)
      }
      if (r.pol == PRESERVE) { r.status = RUNNING; P -= r.kv; A += r.kv; }
      else if (r.pol == SWAP) r.status = SWAPPED;
      else r.status = WAITING;
      r.pend = (int64_t)Rr;
      r.seg = kk + 1;
      r.gen_done = 0;
      F[F_RETURNS]++;
      paused.erase(std::find(paused.begin(), paused.end(), id));
      active.push_back(id);
    }
    // S3 arrivals (Algorithm 1 lines 2-9; Eq.4-15)
    while (next_arr < n && tr.arr_tick[r0 + next_arr] <= t * T) {
      uint32_t id = next_arr++;
      Req& r = R[id];
      uint64_t L = tr.l_pre[r0 + id];
      uint64_t O = tr.gen_pred[seg(id, 0)];
      if (nseg(id) > 1) {
        double Ai = (double)tr.dur_pred[seg(id, 0)];
        int pol = select_policy(k, L + O, Ai, (uint64_t)A_snap, ip.policy_mode);  // R4, R5, R7
        r.V = stage1_value(k, L, O, Ai, pol);
      } else {
        r.V = stage1_value(k, L, O, 0.0, DISCARD);  // no call: Discard form (R11)
      }
      r.status = WAITING;
      r.pend = (int64_t)L;
      r.last = t;                                 // R14, R31
      F[F_ARRIVED]++;
      active.push_back(id);
    }
    // idle check: jump to the next event iteration (not counted)
    if (active.empty()) {
      uint64_t te = UINT64_MAX;
      if (next_arr < n) te = (tr.arr_tick[r0 + next_arr] + T - 1) / T;
      for (uint32_t id : paused) te = std::min(te, (R[id].ret_tick + T - 1) / T);
      if (te == UINT64_MAX) break;
      t = te;
      continue;
    }
    // S4 budget (Eq.27-32 + clamp; Algorithm 1 lines 25-27)
    int64_t B = ip.budget_mode == 1 ? (int64_t)ip.l_static : token_budget(cfg, cap, A, P, bnd);
    // S5 keys (Eq.26 with R1, R3; FCFS: key 0, R33)
    struct Ent { int tier; uint32_t key; uint32_t id; };
    std::vector<Ent> ord;
    ord.reserve(active.size());
    for (uint32_t id : active) {
      const Req& r = R[id];
      int tier = r.status == RUNNING ? 0 : r.status == SWAPPED ? 1 : 2;  // R16
      uint32_t key = order_key(ip, r.V, k.Ts, t, r.last, id);
      ord.push_back({tier, key, id});
    }
    // S6 order: running => swapped => waiting, each by value, ties by id (R2)
    std::sort(ord.begin(), ord.end(), [](const Ent& a, const Ent& b) {
      return std::tie(a.tier, a.key, a.id) < std::tie(b.tier, b.key, b.id);
    });
    // S7 admission: a prefix with a partial chunk (R17)
    std::vector<int64_t> g(ord.size(), 0);
    int64_t Pj = 0;
    for (size_t j = 0; j < ord.size(); ++j) {
      if (Pj >= B) break;
      int64_t d = demand_of(R[ord[j].id], cfg.s_in);
      g[j] = std::min(d, B - Pj);
      Pj += d;
    }
    // S8 memory resolution (R20)
    int64_t need = 0;
    for (int64_t x : g) need += x;
    int64_t free_ = cap - A - P;
    if (need > free_) {
      std::vector<uint32_t> pres;
      for (uint32_t id : paused)
        if (R[id].pol == PRESERVE && R[id].kv > 0) pres.push_back(id);
      std::sort(pres.begin(), pres.end(), [&](uint32_t a, uint32_t b) {
        if (R[a].kv != R[b].kv) return R[a].kv > R[b].kv;   // kv desc
        return a < b;                                      // id asc
      });
      for (uint32_t id : pres) {
        if (need <= free_) break;
        free_ += R[id].kv; P -= R[id].kv; R[id].kv = 0; R[id].pol = DISCARD;
        F[F_DEMOTE]++;
      }
      for (size_t j = ord.size(); j-- > 0 && need > free_;) {
        Req& r = R[ord[j].id];
        if (r.kv + g[j] <= 0) continue;
        free_ += r.kv; A -= r.kv; need -= g[j];
        g[j] = 0; r.kv = 0; r.cpu = 0; r.status = WAITING;
        F[F_EVICT]++;
      }
    }
    // S9 last-scheduled time (R14), S10 engine advance (a8)
    F[F_BUSY]++;
    F[F_DECISIONS] += ord.size();
    F[F_MAXQ] = std::max<uint64_t>(F[F_MAXQ], ord.size());
    std::vector<uint32_t> leave;
    for (size_t j = 0; j < ord.size(); ++j) {
      if (g[j] <= 0) continue;
      uint32_t id = ord[j].id;
      Req& r = R[id];
      int64_t x = g[j];
      const int64_t kv_snap = r.kv;
      r.last = t;
      r.status = RUNNING;
      F[F_TOKENS] += (uint64_t)x;
      F[F_ADMITTED]++;
      if (r.cpu > 0) {                               // swap-in
        r.cpu -= x; r.kv += x; A += x;
      } else if ((r.ctx - r.kv) + r.pend > 0) {      // recompute, then prefill/assimilate
        int64_t rc = std::min(x, r.ctx - r.kv);
        r.kv += rc; A += rc;
        int64_t p = x - rc;
        r.pend -= p; r.ctx += p; r.kv += p; A += p;
      } else {                                       // decode one token
        r.ctx += 1; r.kv += 1; A += 1; r.gen_done += 1;
        if (r.ft < 0) r.ft = (int64_t)t + 1;         // R22
        if (r.gen_done == tr.gen_true[seg(id, r.seg)]) {
          if (r.seg + 1 == nseg(id)) {               // last segment: finish
            A -= r.kv; r.kv = 0; r.status = FINISHED;
            ++n_fin;
            uint64_t arr = tr.arr_tick[r0 + id];
            uint64_t fin = t + 1;
            uint64_t ttft = (uint64_t)r.ft * T - arr;
            uint64_t e2e = fin * T - arr;
            bool ok = ttft < ip.slo_ttft_ticks &&
                      e2e * ip.slo_norm_den < (uint64_t)ip.slo_norm_num * T * r.gen_total;
            bool ok5 = ttft < 5 * ip.slo_ttft_ticks &&
                       e2e * ip.slo_norm_den < 5 * (uint64_t)ip.slo_norm_num * T * r.gen_total;
            F[F_COMPLETED]++;
            F[F_SLO_OK] += ok;
            F[F_SLO_OK5] += ok5;
            F[F_MAKESPAN] = std::max<uint64_t>(F[F_MAKESPAN], fin);
            F[F_SUM_TTFT] += ttft;
            F[F_SUM_E2E] += e2e;
            F[F_SUM_GEN] += r.gen_total;
            res->hist_ttft[hist_bin(ttft)]++;
            res->hist_norm[hist_bin(e2e / r.gen_total)]++;
            if (ft_out) ft_out[id] = r.ft;
            if (fin_out) fin_out[id] = (int64_t)fin;
            leave.push_back(id);
          } else {                                   // issue call k = seg (R13)
            uint32_t kk = r.seg;
            double Ti = (double)tr.dur_pred[seg(id, kk)];
            int pol = select_policy(k, (uint64_t)r.ctx, Ti, (uint64_t)(A_snap - kv_snap),
                                    ip.policy_mode);
            r.pol = pol;
            r.ret_tick = (t + 1) * T + tr.dur_true[seg(id, kk)];
            r.status = PAUSED;
            A -= r.kv;
            if (pol == PRESERVE) { P += r.kv; F[F_CALL_P]++; }
            else if (pol == SWAP) { r.cpu = r.ctx; r.kv = 0; F[F_CALL_S]++; }  // R21
            else { r.kv = 0; F[F_CALL_D]++; }
            leave.push_back(id);
            paused.push_back(id);
          }
        }
      }
    }
    if (!leave.empty()) {
      std::vector<uint32_t> keep;
      for (uint32_t id : active)
        if (R[id].status != FINISHED && R[id].status != PAUSED) keep.push_back(id);
      active.swap(keep);
    }
    if (A < 0 || P < 0 || A + P > cap) F[F_ERR] |= 1;  // ledger invariant (§8(c).4)
    t += 1;                                            // S12
  }
  F[F_FINAL_T] = t;
  // R28 / S:481: requests still unfinished when the run stopped (a W1/W3 run
  // stops at the horizon, max_iters = H / T) are excluded from attainment
  // and counted here
  F[F_INCOMPLETE] = n - n_fin;
}


// ---------------------------------------------------------------------------
// Step mode: the scheduler as a library (augsched_step).  The engine reports
// its events as records; one step = Algorithm 1 lines 2-40 for every
// instance, with the token accounting of the granted batch applied.
// ---------------------------------------------------------------------------
enum { S_EMPTY = 0 };
enum { K_NEW = 1, K_RETURN = 2, K_CALL = 3, K_FINISH = 4, K_IMPORT = 5 };

struct SSlot {
  int status = S_EMPTY;
  int pol = DISCARD;
  double V = 0;
  uint64_t last = 0;
  int64_t ctx = 0, kv = 0, cpu = 0, pend = 0;
};
struct SRec {
  uint32_t kind, id, la, lb, lc, flags, last, ctx, kv, cpu, pend;
  float ta;
};
struct SInst {
  std::vector<SSlot> s;
  int64_t A = 0, P = 0;
  std::vector<SRec> rec;
};
struct OStep {
  OCfg cfg;
  std::vector<OInst> ip;
  uint32_t n_inst = 0, max_active = 0;
  std::vector<SInst> inst;
};

// value of an imported / new / returned request (Stage I or Stage II + final)
double intake_value(const Coef& k, const OInst& ip, bool stage2, int pol, uint64_t la,
                    uint64_t lb, uint64_t lc, double ta, bool has_call, int64_t A_snap) {
  if (!stage2) {
    if (!has_call) return stage1_value(k, la, lb, 0.0, DISCARD);
    int p = select_policy(k, la + lb, ta, (uint64_t)A_snap, ip.policy_mode);
    return stage1_value(k, la, lb, ta, p);
  }
  double V2 = stage2_value(k, la, lb, lc, pol);
  if (!has_call) return V2;
  uint64_t X = la + lb + lc;
  int nx = select_policy(k, X, ta, (uint64_t)A_snap, ip.policy_mode);
  return final_value(k, V2, X, nx, ta);
}

int step_one(OStep& S, uint32_t i, uint64_t now, int64_t* B_out, uint32_t* n_out,
             uint32_t* adm_out, uint32_t* order, uint32_t* grant, uint32_t* keys, uint32_t* tier_off) {
  SInst& I = S.inst[i];
  const OInst& ip = S.ip[i];
  const OCfg& cfg = S.cfg;
  const Coef k = make_coef(cfg, ip.target_max);
  const Bounds bnd = clamp_bounds(cfg, ip.target_max);
  const int64_t cap = cap_tokens(cfg);
  int err = 0;
  // engine events of the previous forward: CALL (issue, R13) and FINISH
  const int64_t A_evt = I.A;
  for (const SRec& r : I.rec) {
    if (r.kind != K_CALL && r.kind != K_FINISH) continue;
    SSlot& s = I.s[r.id];
    if (r.kind == K_FINISH) {
      if (s.status < RUNNING || s.status > WAITING) { err = -4; continue; }
      I.A -= s.kv;
      s = SSlot();
    } else {
      if (s.status != RUNNING || s.cpu != 0 || s.kv != s.ctx || s.pend != 0) { err = -4; continue; }
      int pol = select_policy(k, (uint64_t)s.ctx, (double)r.ta, (uint64_t)(A_evt - s.kv),
                              ip.policy_mode);
      s.pol = pol;
      s.status = PAUSED;
      I.A -= s.kv;
      if (pol == PRESERVE) I.P += s.kv;
      else if (pol == SWAP) { s.cpu = s.ctx; s.kv = 0; }
      else s.kv = 0;
    }
  }
  const int64_t A_snap = I.A;  // S1
  std::vector<SRec> rets, news;
  for (const SRec& r : I.rec) {
    if (r.kind == K_RETURN) rets.push_back(r);
    if (r.kind == K_NEW || r.kind == K_IMPORT) news.push_back(r);
  }
  auto by_id = [](const SRec& a, const SRec& b) { return a.id < b.id; };
  std::stable_sort(rets.begin(), rets.end(), by_id);
  std::stable_sort(news.begin(), news.end(), by_id);
  for (const SRec& r : rets) {  // S2
    SSlot& s = I.s[r.id];
    if (s.status != PAUSED) { err = -4; continue; }
    s.V = intake_value(k, ip, true, s.pol, (uint64_t)s.ctx, r.la, r.lb, (double)r.ta,
                       (r.flags & 1) != 0, A_snap);
    if (s.pol == PRESERVE) { s.status = RUNNING; I.P -= s.kv; I.A += s.kv; }
    else if (s.pol == SWAP) s.status = SWAPPED;
    else s.status = WAITING;
    s.pend = r.la;
  }
  for (const SRec& r : news) {  // S3
    SSlot& s = I.s[r.id];
    if (s.status != S_EMPTY) { err = -4; continue; }
    if (r.kind == K_NEW) {
      s.V = intake_value(k, ip, false, DISCARD, r.la, r.lb, 0, (double)r.ta, (r.flags & 1) != 0,
                         A_snap);
      s.status = WAITING; s.pend = r.la; s.last = now;
    } else {
      int st = (r.flags >> 4) & 7, pol = (r.flags >> 8) & 3;
      bool st2 = (r.flags >> 12) & 1;
      // reading B9: a last-scheduled time in the future is a state violation
      // (Eq.26's wait now - last is a time that has passed, R14/R15)
      if ((uint64_t)r.last > now) { err = -4; continue; }
      s.V = intake_value(k, ip, st2, pol, r.la, r.lb, r.lc, (double)r.ta, (r.flags & 1) != 0,
                         A_snap);
      s.status = st; s.pol = pol; s.last = r.last;
      s.ctx = r.ctx; s.kv = r.kv; s.cpu = r.cpu; s.pend = r.pend;
      if (st == PAUSED && pol == PRESERVE) I.P += s.kv; else I.A += s.kv;
    }
  }
  I.rec.clear();
  // S4 budget
  int64_t B = ip.budget_mode == 1 ? (int64_t)ip.l_static : token_budget(cfg, cap, I.A, I.P, bnd);
  // S5 keys, S6 order
  struct Ent { int tier; uint32_t key; uint32_t id; };
  std::vector<Ent> ord;
  for (uint32_t id = 0; id < S.max_active; ++id) {
    const SSlot& s = I.s[id];
    if (s.status < RUNNING || s.status > WAITING) continue;
    uint32_t key = order_key(ip, s.V, k.Ts, now, s.last, id);
    ord.push_back({s.status - RUNNING, key, id});
  }
  std::sort(ord.begin(), ord.end(), [](const Ent& a, const Ent& b) {
    return std::tie(a.tier, a.key, a.id) < std::tie(b.tier, b.key, b.id);
  });
  // S7 admission
  std::vector<int64_t> g(ord.size(), 0);
  int64_t Pj = 0;
  uint32_t n_prefix = 0;  // admission prefix length (entries with P_{j-1} < B)
  for (size_t j = 0; j < ord.size(); ++j) {
    if (Pj >= B) break;
    ++n_prefix;
    int64_t d;
    const SSlot& s = I.s[ord[j].id];
    if (s.cpu > 0) d = std::min<int64_t>(s.cpu, cfg.s_in);
    else if ((s.ctx - s.kv) + s.pend > 0) d = (s.ctx - s.kv) + s.pend;
    else d = 1;
    g[j] = std::min(d, B - Pj);
    Pj += d;
  }
  // S8 resolution
  int64_t need = 0;
  for (int64_t x : g) need += x;
  int64_t free_ = cap - I.A - I.P;
  if (need > free_) {
    std::vector<uint32_t> pres;
    for (uint32_t id = 0; id < S.max_active; ++id)
      if (I.s[id].status == PAUSED && I.s[id].pol == PRESERVE && I.s[id].kv > 0) pres.push_back(id);
    std::sort(pres.begin(), pres.end(), [&](uint32_t a, uint32_t b) {
      if (I.s[a].kv != I.s[b].kv) return I.s[a].kv > I.s[b].kv;
      return a < b;
    });
    for (uint32_t id : pres) {
      if (need <= free_) break;
      SSlot& s = I.s[id];
      free_ += s.kv; I.P -= s.kv; s.kv = 0; s.pol = DISCARD;
    }
    for (size_t j = ord.size(); j-- > 0 && need > free_;) {
      SSlot& s = I.s[ord[j].id];
      if (s.kv + g[j] <= 0) continue;
      free_ += s.kv; I.A -= s.kv; need -= g[j];
      g[j] = 0; s.kv = 0; s.cpu = 0; s.status = WAITING;
    }
  }
  // S9 + token accounting of the granted batch
  for (size_t j = 0; j < ord.size(); ++j) {
    order[j] = ord[j].id;
    keys[j] = ord[j].key;
    grant[j] = (uint32_t)g[j];
    if (g[j] <= 0) continue;
    SSlot& s = I.s[ord[j].id];
    int64_t x = g[j];
    s.last = now;
    s.status = RUNNING;
    if (s.cpu > 0) { s.cpu -= x; s.kv += x; I.A += x; }
    else if ((s.ctx - s.kv) + s.pend > 0) {
      int64_t rc = std::min(x, s.ctx - s.kv);
      s.kv += rc; I.A += rc;
      int64_t p = x - rc;
      s.pend -= p; s.ctx += p; s.kv += p; I.A += p;
    } else { s.ctx += 1; s.kv += 1; I.A += 1; }
  }
  *B_out = B;
  *n_out = (uint32_t)ord.size();
  *adm_out = n_prefix;
  // tier segment starts of the order (running => swapped => waiting)
  for (int t = 0; t < 3; ++t) {
    uint32_t c = 0;
    for (const Ent& e : ord) c += e.tier < t;
    tier_off[t] = c;
  }
  return err;
}

}  // namespace

// ============================================================================
// C ABI (for ctypes in oracle/__init__.py)
// ============================================================================
extern "C" {

int oracle_simulate(const OCfg* cfg, const OInst* inst, uint32_t n_inst, const OTrace* tr,
                    const uint32_t* inst_trace_id, uint64_t max_iters, OResult* out,
                    int n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::atomic<uint32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      uint32_t i = next.fetch_add(1);
      if (i >= n_inst) break;
      simulate_one(*cfg, inst[i], *tr, inst_trace_id[i], max_iters, &out[i]);
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n_threads; ++i) th.emplace_back(worker);
  worker();
  for (auto& x : th) x.join();
  return 0;
}

// one instance with per-request first-token / finish iterations (-1 = none)
int oracle_simulate_detail(const OCfg* cfg, const OInst* inst, const OTrace* tr, uint32_t trace_id,
                           uint64_t max_iters, OResult* out, int64_t* ft, int64_t* fin) {
  uint32_t n = tr->req_off[trace_id + 1] - tr->req_off[trace_id];
  for (uint32_t i = 0; i < n; ++i) ft[i] = fin[i] = -1;
  simulate_one(*cfg, *inst, *tr, trace_id, max_iters, out, ft, fin);
  return 0;
}

// ---- formula entry points for the pin tests --------------------------------
double oracle_waste(const OCfg* c, uint32_t target_max, int pol, uint64_t C, double Ti,
                    uint64_t Co) {
  Coef k = make_coef(*c, target_max);
  if (pol == PRESERVE) return waste_preserve(k, Ti, C);
  if (pol == SWAP) return waste_swap(k, C);
  return waste_discard(k, C, Co);
}
int oracle_select_policy(const OCfg* c, uint32_t target_max, uint64_t C, double Ti, uint64_t Co,
                         uint32_t policy_mode) {
  return select_policy(make_coef(*c, target_max), C, Ti, Co, policy_mode);
}
double oracle_stage1(const OCfg* c, uint32_t target_max, uint64_t L, uint64_t O, double A,
                     int pol) {
  return stage1_value(make_coef(*c, target_max), L, O, A, pol);
}
double oracle_stage2(const OCfg* c, uint32_t target_max, uint64_t Lt, uint64_t R, uint64_t O,
                     int pol) {
  return stage2_value(make_coef(*c, target_max), Lt, R, O, pol);
}
double oracle_final(const OCfg* c, uint32_t target_max, double V2, uint64_t X, int next_pol,
                    double An) {
  return final_value(make_coef(*c, target_max), V2, X, next_pol, An);
}
uint32_t oracle_key(double V, double alpha, double Ts, uint64_t now, uint64_t last) {
  return sched_key(V, alpha, Ts, now, last);
}
int64_t oracle_budget(const OCfg* c, uint32_t target_max, int64_t A, int64_t P) {
  return token_budget(*c, cap_tokens(*c), A, P, clamp_bounds(*c, target_max));
}
int64_t oracle_cap(const OCfg* c) { return cap_tokens(*c); }
uint64_t oracle_splitmix64_mix(uint64_t z) { return splitmix64_mix(z); }
uint32_t oracle_random_key(uint32_t seed, uint32_t id, uint64_t t) { return random_key(seed, id, t); }
uint32_t oracle_hist_bin(uint64_t v) { return hist_bin(v); }
uint32_t oracle_result_size(void) { return (uint32_t)sizeof(OResult); }

// ---- step mode ---------------------------------------------------------------
void* oracle_step_create(const OCfg* cfg, const OInst* inst, uint32_t n_inst, uint32_t max_active) {
  OStep* S = new OStep();
  S->cfg = *cfg;
  S->ip.assign(inst, inst + n_inst);
  S->n_inst = n_inst;
  S->max_active = max_active;
  S->inst.resize(n_inst);
  for (auto& I : S->inst) I.s.resize(max_active);
  return S;
}
void oracle_step_destroy(void* h) { delete (OStep*)h; }
// records as SoA arrays (see oracle/__init__.py)
int oracle_step_enqueue(void* h, uint32_t inst, uint32_t n, const uint32_t* kind,
                        const uint32_t* id, const uint32_t* la, const uint32_t* lb,
                        const uint32_t* lc, const float* ta, const uint32_t* flags,
                        const uint32_t* last, const uint32_t* ctx, const uint32_t* kv,
                        const uint32_t* cpu, const uint32_t* pend) {
  OStep* S = (OStep*)h;
  if (inst >= S->n_inst) return -1;
  for (uint32_t j = 0; j < n; ++j) {
    if (id[j] >= S->max_active || kind[j] < K_NEW || kind[j] > K_IMPORT) return -1;
    SRec r{kind[j], id[j], la[j], lb[j], lc[j], flags[j], last[j], ctx[j], kv[j], cpu[j], pend[j],
           ta[j]};
    S->inst[inst].rec.push_back(r);
  }
  return 0;
}
int oracle_step(void* h, uint64_t now, int64_t* B, uint32_t* n_active, uint32_t* admitted,
                uint32_t* order, uint32_t* grant, uint32_t* keys, uint32_t* tier_off) {
  OStep* S = (OStep*)h;
  int err = 0;
  for (uint32_t i = 0; i < S->n_inst; ++i) {
    size_t off = (size_t)i * S->max_active;
    int e = step_one(*S, i, now, &B[i], &n_active[i], &admitted[i], order + off, grant + off,
                     keys + off, tier_off + 3 * (size_t)i);
    if (e) err = e;
  }
  return err;
}
// slot state: status (0 empty, 1 run, 2 swap, 3 wait, 4 paused), policy, token counts
void oracle_step_slot(void* h, uint32_t inst, uint32_t id, int32_t* out6) {
  const SSlot& s = ((OStep*)h)->inst[inst].s[id];
  out6[0] = s.status; out6[1] = s.pol; out6[2] = (int32_t)s.ctx; out6[3] = (int32_t)s.kv;
  out6[4] = (int32_t)s.cpu; out6[5] = (int32_t)s.pend;
}
void oracle_step_slots_all(void* h, uint32_t inst, int32_t* out) {   // [max_active][6]
  OStep* S = (OStep*)h;
  for (uint32_t id = 0; id < S->max_active; ++id) oracle_step_slot(h, inst, id, out + 6 * (size_t)id);
}
void oracle_step_ledger(void* h, uint32_t inst, int64_t* A, int64_t* P) {
  OStep* S = (OStep*)h;
  *A = S->inst[inst].A;
  *P = S->inst[inst].P;
}

}  // extern "C"
