"""Counter-based, table-driven workload generator (W1 / W2 / W3).

SURVEY §8(f) f3: the same traces can be drawn on the host (here, numpy) and on
the device (`augsched_generate` in libaugsched), bit for bit, because every
random number is a pure function of (seed, trace, request, field) and every
continuous distribution is sampled through a quantile table built once on
the host:

    u(trace, req, field) = mix(mix(seed << 32 | trace) ^ (req << 12 | field))
    mix = the SplitMix64 output function (z += 0x9E37...; two xor-shift-
          multiply rounds; xor-shift), the same function reading B8 uses
    sample = TABLE[u >> 52]           (4,096-entry quantile table at the
                                       midpoints (i + 0.5) / 4096)

Integer draws use the high 32 bits `h = u >> 32`: a class is the number of
cumulative-share thresholds <= h; U{lo..hi} is lo + ((h * (hi - lo + 1)) >> 32);
a Bernoulli(p) draw is h < floor(p * 2^32).  Floating point appears only in
IEEE-exact single operations (one multiply + rint for the arrival gaps; a
divide, a multiply and one fp32 rounding for the predicted durations), which
numpy and the device compute identically.

Fields of request j of trace k: 0 inter-arrival gap, 1 prompt, 2 tool class,
3 calls, 4 no-call draw; segment s of the request uses fields 16 + 8 s + c:
c = 0 generated tokens, 1 predictor hit, 2 wrong-bucket shift, 3 call
duration, 4 returned tokens, 5 duration-prediction noise.

Arrivals: W1/W2 Poisson (unit-mean exponential gaps), W3 Gamma with
coefficient of variation `cv` (shape 1/cv^2, unit mean); gaps are scaled by
1e6 / rate and rounded to integer microsecond ticks; arrival ticks are their
cumulative sum.  W2 keeps exactly `n_max` requests per trace; W1/W3 keep the
arrivals at or before `horizon_ticks` (30 minutes in the paper).

The distribution parameters are those of tracegen's W2 recipe,
quantised to 4,096 levels; they are invented (the paper's figures are
placeholders).  This module holds no arithmetic of the scheduling method.
"""
from __future__ import annotations

import numpy as np
from scipy import stats

from . import BUCKET_EDGES, BUCKET_MID, TOOL_MIX, Traces, _finish

NQ = 4096                       # quantile-table levels (12 bits of u)
NCLASS = 4
MAXSEG = 255                    # segments per request the simulator accepts
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    """SplitMix64 output function, vectorised over uint64 arrays."""
    with np.errstate(over="ignore"):
        z = (np.asarray(z, np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _u(key_trace, req, field):
    """Uniform u64 of (trace key, request index, field)."""
    return mix64(key_trace ^ ((np.asarray(req, np.uint64) << np.uint64(12)) | np.uint64(field)))


def _q(dist_ppf):
    p = (np.arange(NQ, dtype=np.float64) + 0.5) / NQ
    return dist_ppf(p)


def _lognormal_table(median, sigma, lo, hi):
    x = _q(lambda p: stats.lognorm.ppf(p, sigma, scale=median))
    return np.clip(np.rint(x), lo, hi).astype(np.uint32)


def build_tables(cv: float | None = None, accuracy: float = 0.65, dur_noise_sigma: float = 0.5,
                 p_nocall: float = 0.0, prompt=(400.0, 0.8, 8, 4096), gen=(48.0, 0.9, 1, 1024),
                 tool_mix=None, predictor: str = "bucket") -> dict:
    """Quantile tables and thresholds of one workload recipe (host, once).
    cv=None: Poisson arrivals (W1/W2); cv>0: Gamma arrivals with that CV (W3)."""
    mix = TOOL_MIX if tool_mix is None else tool_mix
    names = list(mix.keys())
    assert len(names) == NCLASS
    if cv is None:
        gap = _q(lambda p: stats.expon.ppf(p))
    else:
        k = 1.0 / (cv * cv)
        gap = _q(lambda p: stats.gamma.ppf(p, k, scale=1.0 / k))
    shares = np.array([mix[n][0] for n in names], np.float64)
    shares = shares / shares.sum()
    th = np.floor(np.cumsum(shares)[:-1] * 2.0**32).astype(np.uint64)
    return dict(
        gap=np.ascontiguousarray(gap, np.float64),
        prompt=_lognormal_table(*prompt),
        gen=_lognormal_table(*gen),
        cls_th=np.ascontiguousarray(th.astype(np.uint32)),
        calls_lo=np.array([mix[n][1] for n in names], np.uint32),
        calls_hi=np.array([mix[n][2] for n in names], np.uint32),
        dur=np.stack([_lognormal_table(mix[n][3] * 1e6, mix[n][4], 1, 2**31) for n in names]),
        ret=np.stack([_lognormal_table(mix[n][5], mix[n][6], mix[n][7], mix[n][8]) for n in names]),
        noise=np.ascontiguousarray(_q(lambda p: stats.lognorm.ppf(p, dur_noise_sigma)), np.float64),
        edges=np.ascontiguousarray(BUCKET_EDGES, np.uint32),
        mids=np.ascontiguousarray(BUCKET_MID, np.uint32),
        acc_th=np.uint32(min(int(np.floor(accuracy * 2.0**32)), 2**32 - 1)),
        nocall_th=np.uint32(min(int(np.floor(p_nocall * 2.0**32)), 2**32 - 1)),
        oracle_pred=np.uint32(1 if predictor == "oracle" else 0),
    )


def generate(tables: dict, seed: int, n_traces: int, n_max: int, rates, horizon_ticks: int = 0) -> Traces:
    """Host reference of the counter-based generator: `n_traces` traces of up
    to `n_max` requests, trace k at rates[k % len(rates)] req/s; horizon 0 =
    W2 (exactly n_max requests), else W1/W3 (arrivals <= horizon)."""
    rates = list(rates) if hasattr(rates, "__len__") else [rates]
    T = tables
    parts = []
    counts = []
    for k in range(n_traces):
        kt = mix64(np.uint64((int(seed) << 32) | k))
        j = np.arange(n_max, dtype=np.uint64)
        scale = 1e6 / float(rates[k % len(rates)])
        gap = np.rint(T["gap"][(_u(kt, j, 0) >> np.uint64(52)).astype(np.int64)] * scale)
        arr = np.cumsum(gap.astype(np.uint64))
        n = n_max if horizon_ticks == 0 else int(np.searchsorted(arr, np.uint64(horizon_ticks), side="right"))
        j = j[:n]
        arr = arr[:n]
        lpre = T["prompt"][(_u(kt, j, 1) >> np.uint64(52)).astype(np.int64)]
        h2 = (_u(kt, j, 2) >> np.uint64(32))
        cls = np.zeros(n, np.int64)
        for t in T["cls_th"]:
            cls += (h2 >= np.uint64(t)).astype(np.int64)
        lo = T["calls_lo"][cls].astype(np.uint64)
        span = T["calls_hi"][cls].astype(np.uint64) - lo + np.uint64(1)
        with np.errstate(over="ignore"):
            calls = lo + (((_u(kt, j, 3) >> np.uint64(32)) * span) >> np.uint64(32))
        nocall = (_u(kt, j, 4) >> np.uint64(32)) < np.uint64(T["nocall_th"])
        calls = np.where(nocall, np.uint64(0), calls)
        nseg = (calls + np.uint64(1)).astype(np.int64)
        assert int(nseg.max(initial=1)) <= MAXSEG
        # segments, request-major
        rq = np.repeat(j, nseg)
        sk = np.concatenate([np.arange(s, dtype=np.uint64) for s in nseg]) if n else np.zeros(0, np.uint64)
        scls = np.repeat(cls, nseg)
        last = np.zeros(sk.shape[0], bool)
        if n:
            last[np.cumsum(nseg) - 1] = True
        fb = np.uint64(16) + np.uint64(8) * sk
        gen_t = T["gen"][(_u(kt, rq, fb + np.uint64(0)) >> np.uint64(52)).astype(np.int64)]
        if T["oracle_pred"]:
            gen_p = gen_t.copy()
        else:
            b = np.searchsorted(T["edges"], gen_t, side="right") - 1
            hit = (_u(kt, rq, fb + np.uint64(1)) >> np.uint64(32)) < np.uint64(T["acc_th"])
            with np.errstate(over="ignore"):
                shift = np.uint64(1) + (((_u(kt, rq, fb + np.uint64(2)) >> np.uint64(32)) * np.uint64(7))
                                        >> np.uint64(32))
            b2 = np.where(hit, b, (b + shift.astype(np.int64)) % 8)
            gen_p = T["mids"][b2]
        didx = (_u(kt, rq, fb + np.uint64(3)) >> np.uint64(52)).astype(np.int64)
        dur_t = np.where(last, 0, T["dur"][scls, didx]).astype(np.uint32)
        ridx = (_u(kt, rq, fb + np.uint64(4)) >> np.uint64(52)).astype(np.int64)
        ret = np.where(last, 0, T["ret"][scls, ridx]).astype(np.uint32)
        if T["oracle_pred"]:
            dur_p = (dur_t.astype(np.float64) / 1e6).astype(np.float32)
        else:
            noise = T["noise"][(_u(kt, rq, fb + np.uint64(5)) >> np.uint64(52)).astype(np.int64)]
            dur_p = (dur_t.astype(np.float64) / 1e6 * noise).astype(np.float32)
        dur_p[last] = 0.0
        parts.append((arr, lpre, nseg, gen_t, gen_p, dur_t, dur_p, ret))
        counts.append(n)
    req_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(8)]
    return _finish(req_off, *cat)
