"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the scheduling method (no costs, values,
wastes, budgets or keys).  It only draws workloads: arrival ticks, lengths,
tool-call durations/return lengths and the predictor stand-ins, as flat
numpy arrays (CSR SoA).  Both `oracle/` and `paper_2512_04013_b200/` consume
these arrays; neither imports the other.

Workload recipe (SURVEY.md §8(d) "Synthetic workload (G1)"
W2 = fixed request count with Poisson arrivals; the tool mix and every
distribution parameter below are invented because the paper's figures are
[FIGURE] placeholders):

* arrivals   : cumulative sum of round(1e6 * Exp(rate)) integer µs ticks.
* prompt     : log-normal(median 400, sigma 0.8) clamped to [8, 4096].
* gen/segment: log-normal(median 48, sigma 0.9) clamped to [1, 1024].
* tool class : math 0.25 / QA 0.30 / web 0.25 / chatbot 0.20 with calls per
  request U{1..4}/U{1..3}/U{1..3}/U{2..5}; call duration and return length
  log-normal per class (table in SURVEY §8(d)); optional share of requests
  with no call (`p_nocall`, default 0).
* predictors : output length by a bucket classifier (edges
  1/16/32/64/128/256/512/1024, accuracy 0.65 = the Merge level; the
  reported value is the bucket midpoint); durations by
  multiplicative log-normal noise exp(N(0, 0.5^2)).  predictor="oracle"
  reports the truth (used for the hand-worked goldens).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

# --------------------------------------------------------------------------
# Trace container (CSR over traces -> requests -> segments)
# --------------------------------------------------------------------------


@dataclass
class Traces:
    """Flat SoA trace set.

    req_off[n_traces+1]  u32  request range of each trace
    arr_tick[n_req]      u64  arrival time, integer µs ticks (nondecreasing per trace)
    l_pre[n_req]         u32  prompt tokens (L^pre)
    seg_off[n_req]       u32  first segment index of the request
    n_seg[n_req]         u32  number of segments (calls = n_seg - 1)
    gen_true[n_segs]     u32  tokens decoded in the segment (>= 1)
    gen_pred[n_segs]     u32  predicted tokens for the segment (L^out hat)
    dur_true[n_segs]     u32  true call duration after the segment, µs (0 for last)
    dur_pred[n_segs]     f32  predicted call duration, seconds (T^api hat)
    ret_len[n_segs]      u32  tokens returned by the call (0 for last)
    """

    req_off: np.ndarray
    arr_tick: np.ndarray
    l_pre: np.ndarray
    seg_off: np.ndarray
    n_seg: np.ndarray
    gen_true: np.ndarray
    gen_pred: np.ndarray
    dur_true: np.ndarray
    dur_pred: np.ndarray
    ret_len: np.ndarray

    @property
    def n_traces(self) -> int:
        return int(self.req_off.shape[0] - 1)

    @property
    def n_req(self) -> int:
        return int(self.arr_tick.shape[0])

    def trace_len(self, i: int) -> int:
        return int(self.req_off[i + 1] - self.req_off[i])

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in (
            "req_off", "arr_tick", "l_pre", "seg_off", "n_seg", "gen_true",
            "gen_pred", "dur_true", "dur_pred", "ret_len")}

    def nbytes(self) -> int:
        return int(sum(a.nbytes for a in self.arrays().values()))


def _finish(req_off, arr, lpre, nseg, gen_t, gen_p, dur_t, dur_p, ret) -> Traces:
    nseg = np.asarray(nseg, np.uint32)
    seg_off = np.zeros(nseg.shape[0], np.uint32)
    if nseg.shape[0] > 1:
        seg_off[1:] = np.cumsum(nseg[:-1], dtype=np.uint64).astype(np.uint32)
    return Traces(
        req_off=np.ascontiguousarray(req_off, np.uint32),
        arr_tick=np.ascontiguousarray(arr, np.uint64),
        l_pre=np.ascontiguousarray(lpre, np.uint32),
        seg_off=seg_off,
        n_seg=nseg,
        gen_true=np.ascontiguousarray(gen_t, np.uint32),
        gen_pred=np.ascontiguousarray(gen_p, np.uint32),
        dur_true=np.ascontiguousarray(dur_t, np.uint32),
        dur_pred=np.ascontiguousarray(dur_p, np.float32),
        ret_len=np.ascontiguousarray(ret, np.uint32),
    )


# --------------------------------------------------------------------------
# Hand-built traces (goldens) — list of dicts
# --------------------------------------------------------------------------


def from_requests(traces: list[list[dict]]) -> Traces:
    """Build a Traces object from explicit request dicts.

    Each request: {"arr": ticks, "l_pre": L, "segs": [(gen_true, gen_pred,
    dur_true_ticks, dur_pred_s, ret_len), ...]} — the last segment's call
    fields are ignored (set to 0).
    """
    req_off = [0]
    arr, lpre, nseg = [], [], []
    gt, gp, dt, dp, rl = [], [], [], [], []
    for tr in traces:
        for r in tr:
            arr.append(int(r["arr"]))
            lpre.append(int(r["l_pre"]))
            segs = r["segs"]
            nseg.append(len(segs))
            for k, s in enumerate(segs):
                g_true, g_pred = int(s[0]), int(s[1])
                last = k == len(segs) - 1
                gt.append(g_true)
                gp.append(g_pred)
                dt.append(0 if last else int(s[2]))
                dp.append(0.0 if last else float(s[3]))
                rl.append(0 if last else int(s[4]))
        req_off.append(len(arr))
    return _finish(req_off, arr, lpre, nseg, gt, gp, dt, dp, rl)


# --------------------------------------------------------------------------
# Synthetic W2 generator
# --------------------------------------------------------------------------

# (share, calls lo, calls hi, dur median s, dur sigma, ret median, ret sigma, ret lo, ret hi)
TOOL_MIX = {
    "math":    (0.25, 1, 4, 0.01, 0.5, 8.0, 0.5, 1, 64),
    "qa":      (0.30, 1, 3, 0.7, 0.6, 200.0, 0.8, 16, 2048),
    "web":     (0.25, 1, 3, 2.0, 0.8, 600.0, 0.8, 32, 4096),
    "chatbot": (0.20, 2, 5, 20.0, 0.7, 40.0, 0.6, 4, 512),
}
BUCKET_EDGES = np.array([1, 16, 32, 64, 128, 256, 512, 1024], np.int64)
BUCKET_MID = np.array([8, 24, 48, 96, 192, 384, 768, 1024], np.int64)


def _lognormal_int(rng, median, sigma, lo, hi, size):
    x = rng.lognormal(np.log(median), sigma, size)
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


def _bucket_predict(rng, truth, accuracy):
    b = np.searchsorted(BUCKET_EDGES, truth, side="right") - 1
    b = np.clip(b, 0, len(BUCKET_EDGES) - 1)
    wrong = rng.random(truth.shape[0]) >= accuracy
    # uniformly chosen wrong bucket
    shift = rng.integers(1, len(BUCKET_EDGES), truth.shape[0])
    b2 = np.where(wrong, (b + shift) % len(BUCKET_EDGES), b)
    return BUCKET_MID[b2]


def gen_trace_arrays(n: int, rate: float, seed: int, trace_id: int = 0,
                     predictor: str = "bucket", accuracy: float = 0.65,
                     dur_noise_sigma: float = 0.5, p_nocall: float = 0.0,
                     prompt=(400.0, 0.8, 8, 4096), gen=(48.0, 0.9, 1, 1024),
                     tool_mix=None):
    """One W2 trace of `n` requests at Poisson `rate` req/s."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, trace_id])))
    mix = TOOL_MIX if tool_mix is None else tool_mix
    inter = np.rint(rng.exponential(1.0 / rate, n) * 1e6).astype(np.int64)
    arr = np.cumsum(inter).astype(np.uint64)
    lpre = _lognormal_int(rng, prompt[0], prompt[1], prompt[2], prompt[3], n)
    names = list(mix.keys())
    shares = np.array([mix[k][0] for k in names], np.float64)
    shares = shares / shares.sum()
    cls = rng.choice(len(names), size=n, p=shares)
    ncalls = np.zeros(n, np.int64)
    for ci, name in enumerate(names):
        _, lo, hi = mix[name][:3]
        m = cls == ci
        ncalls[m] = rng.integers(lo, hi + 1, int(m.sum()))
    if p_nocall > 0:
        ncalls[rng.random(n) < p_nocall] = 0
    nseg = ncalls + 1
    tot = int(nseg.sum())
    gen_t = _lognormal_int(rng, gen[0], gen[1], gen[2], gen[3], tot)
    # per-segment class and "is a call" flag
    seg_cls = np.repeat(cls, nseg)
    seg_start = np.concatenate([[0], np.cumsum(nseg)[:-1]])
    is_last = np.zeros(tot, bool)
    is_last[seg_start + nseg - 1] = True
    dur_s = np.zeros(tot, np.float64)
    ret = np.zeros(tot, np.int64)
    for ci, name in enumerate(names):
        _, _, _, dm, ds, rm, rs, rlo, rhi = mix[name]
        m = (seg_cls == ci) & ~is_last
        k = int(m.sum())
        dur_s[m] = rng.lognormal(np.log(dm), ds, k)
        ret[m] = _lognormal_int(rng, rm, rs, rlo, rhi, k)
    dur_t = np.rint(dur_s * 1e6).astype(np.int64)
    dur_t = np.minimum(dur_t, 2**31)
    if predictor == "oracle":
        gen_p = gen_t.copy()
        dur_p = (dur_t.astype(np.float64) / 1e6).astype(np.float32)
    elif predictor == "bucket":
        gen_p = _bucket_predict(rng, gen_t, accuracy)
        noise = np.exp(rng.normal(0.0, dur_noise_sigma, tot))
        dur_p = (dur_t.astype(np.float64) / 1e6 * noise).astype(np.float32)
    else:
        raise ValueError(predictor)
    dur_p[is_last] = 0.0
    dur_t[is_last] = 0
    ret[is_last] = 0
    return arr, lpre, nseg, gen_t, gen_p, dur_t, dur_p, ret


def gen_traces(n_traces: int, n: int, rates, seed: int, **kw) -> Traces:
    """`n_traces` independent W2 traces; trace i uses rates[i % len(rates)]
    and seed stream (seed, i)."""
    rates = list(rates) if hasattr(rates, "__len__") else [rates]
    parts = [gen_trace_arrays(n, rates[i % len(rates)], seed, i, **kw)
             for i in range(n_traces)]
    req_off = np.arange(n_traces + 1, dtype=np.int64) * n
    cat = [np.concatenate([p[j] for p in parts]) for j in range(8)]
    return _finish(req_off, *cat)


def subset(tr: Traces, ids) -> Traces:
    """Traces restricted to trace indices `ids` (renumbered 0..len-1)."""
    arr, lpre, nseg, gt, gp, dt, dp, rl = [], [], [], [], [], [], [], []
    req_off = [0]
    for i in ids:
        a, b = int(tr.req_off[i]), int(tr.req_off[i + 1])
        arr.append(tr.arr_tick[a:b]); lpre.append(tr.l_pre[a:b]); nseg.append(tr.n_seg[a:b])
        if b > a:
            s0 = int(tr.seg_off[a]); s1 = int(tr.seg_off[b - 1] + tr.n_seg[b - 1])
        else:
            s0 = s1 = 0
        gt.append(tr.gen_true[s0:s1]); gp.append(tr.gen_pred[s0:s1]); dt.append(tr.dur_true[s0:s1])
        dp.append(tr.dur_pred[s0:s1]); rl.append(tr.ret_len[s0:s1])
        req_off.append(req_off[-1] + (b - a))
    c = lambda xs: np.concatenate(xs) if xs else np.zeros(0)
    return _finish(req_off, c(arr), c(lpre), c(nseg), c(gt), c(gp), c(dt), c(dp), c(rl))


# --------------------------------------------------------------------------
# Cost-model presets and per-instance parameter sweeps (config values only)
# --------------------------------------------------------------------------

# SURVEY §8(d) "Cost-model presets".  M = GPT-J-6B fp16 KV bytes/token
# (2*28*4096*2); G_total = RTX 4090 24 GiB; target_max = 500 (best
# static limit in tab:maxbatch); t_fwd, S_in/S_out, G_runtime,
# G_safety and alpha are invented.
PRESET_7B = dict(
    m_per_token=458752,
    g_total=24 * 2**30,
    g_model=12_100_000_000,
    g_runtime=2**30,
    g_safety=512 * 2**20,
    t_fwd_ticks=50_000,
    s_in=2048,
    s_out=2048,
    beta_low=0.5,
    beta_high=1.5,
    gamma_num=1,
    gamma_den=1,
)
INST_7B = dict(
    target_max=500,
    l_static=500,
    alpha=100.0 * 458752,
    slo_ttft_ticks=1_000_000,
    slo_norm_num=10,
    slo_norm_den=1,
    ranking=0,       # 0 = AugServe two-stage values, 1 = FCFS, 2 = random
    budget_mode=0,   # 0 = dynamic (Eq.27-32 + clamp), 1 = static l_static
    policy_mode=0,   # 0 = adaptive argmin, 1/2/3 = forced Preserve/Swap/Discard
    rank_seed=0,     # seed of random scheduling
)

# Hand-worked goldens' system: M = 1, T = 0.1 s, N = 50, S_in = S_out = 200
# (SURVEY §8(c).3 cfg0).  g_* chosen so cap = g_total - fixed.
PRESET_G0 = dict(
    m_per_token=1,
    g_total=1_000_000 + 1000,
    g_model=1000,
    g_runtime=0,
    g_safety=0,
    t_fwd_ticks=100_000,
    s_in=200,
    s_out=200,
    beta_low=0.5,
    beta_high=1.5,
    gamma_num=1,
    gamma_den=1,
)
INST_G0 = dict(
    target_max=50, l_static=100, alpha=0.0, slo_ttft_ticks=1_000_000,
    slo_norm_num=10, slo_norm_den=1, ranking=0, budget_mode=1, policy_mode=0, rank_seed=0,
)


def inst_params(n: int, base: dict | None = None, **overrides) -> dict:
    """Per-instance parameter arrays (length n) from a base dict; each
    override may be a scalar or a length-n sequence."""
    base = dict(INST_7B if base is None else base)
    out = {}
    dt = dict(target_max=np.uint32, l_static=np.uint32, alpha=np.float64,
              slo_ttft_ticks=np.uint64, slo_norm_num=np.uint32, slo_norm_den=np.uint32,
              ranking=np.uint32, budget_mode=np.uint32, policy_mode=np.uint32, rank_seed=np.uint32)
    for k, t in dt.items():
        v = overrides.get(k, base.get(k, 0))
        a = np.asarray(v, dtype=t)
        out[k] = np.ascontiguousarray(np.broadcast_to(a, (n,)).astype(t))
    return out


def cfg3_params():
    """Config 3: 64 target_max values {64, 96, ..., 2080} x 64 TTFT SLOs
    0.25*32^(k/63) s, 4,096 instances on one trace."""
    tm = np.arange(64, 2081, 32, dtype=np.uint32)
    assert tm.shape[0] == 64
    slo = np.rint(0.25 * 32.0 ** (np.arange(64) / 63.0) * 1e6).astype(np.uint64)
    TM, SL = np.meshgrid(tm, slo, indexing="ij")
    n = 64 * 64
    return inst_params(n, target_max=TM.ravel(), l_static=TM.ravel(), slo_ttft_ticks=SL.ravel())


def cfg5_params(n_inst: int = 65536):
    """Config 5: 4,096 traces x 16 parameter points (4 target_max x 4 alpha)."""
    tms = np.array([250, 500, 750, 1000], np.uint32)
    als = np.array([0.0, 10.0, 100.0, 1000.0]) * 458752
    k = np.arange(n_inst) % 16
    return inst_params(n_inst, target_max=tms[k // 4], l_static=tms[k // 4], alpha=als[k % 4])


def cfg5_trace_ids(n_inst: int = 65536):
    return (np.arange(n_inst) // 16).astype(np.uint32)


# --------------------------------------------------------------------------
# Config 4: one huge queue, as IMPORT records of augsched_step (input state)
# --------------------------------------------------------------------------

# Ample KV memory for the 1M-request queue (cap ~ 2.2e9 tokens), so the
# limit stays at the clamp hi = 1.5 * 500 = 750 over the benchmark's steps.
PRESET_CFG4 = dict(PRESET_7B, g_total=2**60)

K_IMPORT = 5
ST_RUN, ST_SWAP, ST_WAIT, ST_PAUSED = 1, 2, 3, 4
POL_P, POL_S, POL_D = 0, 1, 2


def cfg4_records(n: int = 1_000_000, seed: int = 4, t0: int = 65536, n_running: int = 512,
                 n_swapped: int = 512, n_paused: int = 16, stage2_share: float = 0.2) -> dict:
    """SoA IMPORT records for a single queue of n slots:
    `n_running` running (Preserve returns, decode-ready: demand 1),
    `n_swapped` swapped (Swap returns: swap-in pending), `n_paused`
    Preserve-paused (hold the ledger's P), and waiting requests: 80% fresh
    (Stage I, prefill pending) and 20% returned Discard (Stage II, recompute
    + assimilation pending).  last = t0 - U{0..65535}.  Features come from
    the W2 generator; the applied policies are assigned, not computed."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 4])))
    arr, lpre, nseg, gt, gp, dt, dp, ret = gen_trace_arrays(n, 4.0, seed, 0)
    s0 = np.concatenate([[0], np.cumsum(nseg)[:-1]])
    L = lpre.astype(np.int64)
    g0, gp0, dp0, r0 = gt[s0].astype(np.int64), gp[s0], dp[s0], ret[s0].astype(np.int64)
    has2 = nseg >= 2
    gp1 = np.where(has2, gp[np.minimum(s0 + 1, len(gp) - 1)], 0)
    dp1 = np.where(nseg >= 3, dp[np.minimum(s0 + 1, len(dp) - 1)], 0.0).astype(np.float32)
    Lt = L + g0
    kind = np.full(n, K_IMPORT, np.uint32)
    status = np.full(n, ST_WAIT, np.int64)
    pol = np.full(n, POL_D, np.int64)
    stage2 = np.zeros(n, np.int64)
    la, lb, lc = L.copy(), gp0.astype(np.int64), np.zeros(n, np.int64)
    ta = dp0.astype(np.float32)
    flag0 = (nseg > 1).astype(np.int64)
    ctx = np.zeros(n, np.int64); kv = np.zeros(n, np.int64)
    cpu = np.zeros(n, np.int64); pend = L.copy()
    idx = rng.permutation(n)
    a, b, c = n_running, n_running + n_swapped, n_running + n_swapped + n_paused
    run, swp, psd, rest = idx[:a], idx[a:b], idx[b:c], idx[c:]
    st2 = rest[rng.random(rest.shape[0]) < stage2_share]
    for grp, st, pl in ((run, ST_RUN, POL_P), (swp, ST_SWAP, POL_S), (psd, ST_PAUSED, POL_P), (st2, ST_WAIT, POL_D)):
        status[grp] = st; pol[grp] = pl; stage2[grp] = 1
        la[grp], lb[grp], lc[grp] = Lt[grp], r0[grp], gp1[grp]
        ta[grp] = dp1[grp]
        flag0[grp] = (nseg[grp] >= 3).astype(np.int64)
    ctx[run] = kv[run] = Lt[run] + r0[run]; pend[run] = 0
    ctx[swp] = Lt[swp]; cpu[swp] = Lt[swp]; pend[swp] = r0[swp]
    ctx[psd] = kv[psd] = Lt[psd]; pend[psd] = 0
    ctx[st2] = Lt[st2]; pend[st2] = r0[st2]
    last = t0 - rng.integers(0, 65536, n)
    flags = flag0 | (status << 4) | (pol << 8) | (stage2 << 12)
    u = lambda x: np.ascontiguousarray(x, np.uint32)
    return dict(kind=kind, id=u(np.arange(n)), la=u(la), lb=u(lb), lc=u(lc), ta=np.ascontiguousarray(ta),
                flags=u(flags), last=u(last), ctx=u(ctx), kv=u(kv), cpu=u(cpu), pend=u(pend))
