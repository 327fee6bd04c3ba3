"""Pins of the oracle's formulas (Eq.4-32) against values the paper / SPEC fix.

Goldens: tests/golden/spec_core_examples.json (SPEC S:97-161, S:293-296 as
re-verified in SURVEY §8(c).3 G1-G2).  Plus closed forms, special cases and
properties that a dropped term, a wrong sign or a swapped operand would break.
"""
import json
import math
import os
import struct

import numpy as np
import pytest

import oracle
from oracle import PRESERVE, SWAP, DISCARD

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_core_examples.json")))
POL = {"P": PRESERVE, "S": SWAP, "D": DISCARD}

# SPEC core-model cfg: M=1, t_fwd=0.1 s, n_fwd_max=50, s_out=s_in=200
CFG = dict(m_per_token=1, g_total=10**9, g_model=1, g_runtime=0, g_safety=0,
           t_fwd_ticks=100_000, s_in=200, s_out=200, gamma_num=1, gamma_den=1,
           beta_low=0.5, beta_high=1.5)
N = 50


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


@pytest.mark.parametrize("ex", G["waste"], ids=lambda e: e["cite"])
def test_waste_spec(ex):
    v = oracle.waste(CFG, N, POL[ex["policy"]], ex["C"], ex["Ti"], ex["Co"])
    assert rel(v, ex["value"]) < 1e-12


@pytest.mark.parametrize("ex", G["select_policy"], ids=lambda e: e["cite"])
def test_select_policy_spec(ex):
    assert oracle.select_policy(CFG, N, ex["C"], ex["Ti"], ex["Co"]) == POL[ex["policy"]]


@pytest.mark.parametrize("ex", G["stage1"], ids=lambda e: e["cite"])
def test_stage1_spec(ex):
    v = oracle.stage1(CFG, N, ex["L"], ex["O"], ex["A"], POL[ex["policy"]])
    assert rel(v, ex["value"]) < 1e-12


@pytest.mark.parametrize("ex", G["stage2"], ids=lambda e: e["cite"])
def test_stage2_spec(ex):
    v = oracle.stage2(CFG, N, ex["Lt"], ex["R"], ex["O"], POL[ex["policy"]])
    assert rel(v, ex["value"]) < 1e-12


@pytest.mark.parametrize("ex", G["final"], ids=lambda e: e["cite"])
def test_final_spec(ex):
    v = oracle.final(CFG, N, ex["V2"], ex["X"], POL[ex["next"]], ex["An"])
    assert rel(v, ex["value"]) < 1e-12


def f32_key(x):
    u = struct.unpack("<I", struct.pack("<f", x))[0]
    return (~u & 0xFFFFFFFF) if (u & 0x80000000) else (u | 0x80000000)


@pytest.mark.parametrize("ex", G["priority"], ids=lambda e: e["cite"])
def test_priority_spec(ex):
    # wait of 10 s at T = 0.1 s is 100 iterations (R15)
    Ts = 0.1
    now, last = int(round(ex["wait_s"] / Ts)), 0
    k = oracle.key(ex["V"], ex["alpha"], Ts, now, last)
    assert k == f32_key(ex["score"])


@pytest.mark.parametrize("case", G["budget"]["cases"], ids=lambda e: e["cite"])
def test_budget_spec(case):
    cfg = dict(CFG, g_total=1000, g_model=400, g_runtime=0, g_safety=0)
    assert oracle.cap(cfg) == 600
    assert oracle.budget(cfg, 300, case["A"], case["P"]) == case["B"]


# ---------------------------------------------------------------- stage II components
def test_stage2_components_closed_form():
    """swap-in 3.025, recompute 12.1, pro-api 4.8, decode-post 66.25.
    Differences of the three policies isolate each component (Eq.20-22)."""
    P = oracle.stage2(CFG, N, 110, 20, 5, PRESERVE)
    S = oracle.stage2(CFG, N, 110, 20, 5, SWAP)
    D = oracle.stage2(CFG, N, 110, 20, 5, DISCARD)
    assert rel(S - P, 3.025) < 1e-12
    assert rel(D - P, 12.1) < 1e-12
    # pro-api alone: O' = 0 removes decode-post (Eq.19 has no constant term)
    assert rel(oracle.stage2(CFG, N, 110, 20, 0, PRESERVE), 4.8) < 1e-12
    # decode-post alone: R = 0 removes pro-api (Eq.18); Lt+R = 110 -> 0.1*(550+12.5)
    assert rel(oracle.stage2(CFG, N, 110, 0, 5, PRESERVE), 0.1 * (550 + 12.5)) < 1e-12


def test_stage1_scaling_laws():
    """Eq.9-12 are homogeneous: every cost is linear in M; prefill ~ L^2/N."""
    c2 = dict(CFG, m_per_token=2)
    for pol in (PRESERVE, SWAP, DISCARD):
        a = oracle.stage1(CFG, N, 37, 11, 1.5, pol)
        b = oracle.stage1(c2, N, 37, 11, 1.5, pol)
        assert rel(b, 2 * a) < 1e-12
    # O = 0 and Discard leaves prefill only: 1/2 M L^2 / N * T
    assert rel(oracle.stage1(CFG, N, 100, 0, 0.0, DISCARD), 0.5 * 100 * 100 / 50 * 0.1) < 1e-12
    # doubling N halves prefill
    assert rel(oracle.stage1(CFG, 2 * N, 100, 0, 0.0, DISCARD),
               0.5 * oracle.stage1(CFG, N, 100, 0, 0.0, DISCARD)) < 1e-12
    # Preserve - Discard = api = M (L+O) A  (Eq.11)
    d = oracle.stage1(CFG, N, 100, 10, 3.0, PRESERVE) - oracle.stage1(CFG, N, 100, 10, 3.0, DISCARD)
    assert rel(d, 110 * 3.0) < 1e-12


def test_waste_ceiling_and_swap_multiplier():
    """R6: T^fwd(C) = ceil(C/N) T; Eq.6 keeps the N^fwd_max multiplier."""
    # C = 50 -> 1 iteration, C = 51 -> 2 iterations
    assert rel(oracle.waste(CFG, N, DISCARD, 50, 0, 0), 0.1 * 50) < 1e-12
    assert rel(oracle.waste(CFG, N, DISCARD, 51, 0, 0), 0.2 * 51) < 1e-12
    # swap waste doubles when N doubles
    assert rel(oracle.waste(CFG, 2 * N, SWAP, 100, 0, 0), 2 * oracle.waste(CFG, N, SWAP, 100, 0, 0)) < 1e-12


def test_policy_argmin_property():
    """Eq.7-8: the selected waste equals the min of the three, with
    ties Preserve > Swap > Discard (R8)."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        C_ = int(rng.integers(0, 3000))
        Ti = float(np.float32(rng.choice([0.0, rng.exponential(1.0)])))
        Co = int(rng.integers(0, 30000))
        w = [oracle.waste(CFG, N, p, C_, Ti, Co) for p in (PRESERVE, SWAP, DISCARD)]
        p = oracle.select_policy(CFG, N, C_, Ti, Co)
        assert w[p] == min(w)
        assert p == [i for i in range(3) if w[i] == min(w)][0]
    for pm, want in ((1, PRESERVE), (2, SWAP), (3, DISCARD)):
        assert oracle.select_policy(CFG, N, 100, 2.0, 300, pm) == want


def test_values_nonnegative_and_monotone():
    """costs are nonnegative; Stage I nondecreasing in L, O, A."""
    rng = np.random.default_rng(1)
    for _ in range(500):
        L, O = int(rng.integers(1, 4000)), int(rng.integers(0, 1000))
        A = float(rng.exponential(2.0))
        for pol in (PRESERVE, SWAP, DISCARD):
            v = oracle.stage1(CFG, N, L, O, A, pol)
            assert v >= 0
            assert oracle.stage1(CFG, N, L + 1, O, A, pol) >= v
            assert oracle.stage1(CFG, N, L, O + 1, A, pol) >= v
        assert oracle.stage1(CFG, N, L, O, A + 1.0, PRESERVE) >= oracle.stage1(CFG, N, L, O, A, PRESERVE)
        for pol in (PRESERVE, SWAP, DISCARD):
            assert oracle.stage2(CFG, N, L, O, int(rng.integers(0, 500)), pol) >= 0


# ---------------------------------------------------------------- key (R1, R3)
def test_key_order_matches_float_order():
    """orderable-u32 of fp32 is monotone in the float value (numpy's float32
    ordering is the independent reference)."""
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.normal(0, 1e9, 2000), rng.normal(0, 1, 2000), [0.0, 1.0, -1.0, 3e38, -3e38]])
    keys = np.array([oracle.key(float(v), 0.0, 0.1, 0, 0) for v in x], np.uint64)
    f = x.astype(np.float32)
    o1 = np.lexsort((np.arange(len(f)), f))
    o2 = np.lexsort((np.arange(len(f)), keys))
    assert np.array_equal(f[o1], f[o2])


def test_key_is_single_rounding_of_double_score():
    """s = V - alpha*w in binary64 then one RN to fp32 (R3): compare with numpy
    scalar float64 arithmetic (IEEE, no contraction)."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        V = float(rng.uniform(0, 1e10))
        alpha = float(rng.choice([0.0, 458752.0 * 100]))
        now = int(rng.integers(0, 100000))
        last = int(rng.integers(0, now + 1))
        Ts = 0.05
        s = np.float64(V) - np.float64(alpha) * (np.float64(now - last) * np.float64(Ts))
        assert oracle.key(V, alpha, Ts, now, last) == f32_key(float(np.float32(s)))


def test_anti_starvation_sign():
    """R1: waiting lowers the score (raises priority)."""
    k0 = oracle.key(100.0, 2.0, 0.1, 0, 0)
    k1 = oracle.key(100.0, 2.0, 0.1, 50, 0)
    assert k1 < k0


# ---------------------------------------------------------------- budget (Eq.27-32)
def test_budget_properties():
    cfg = dict(CFG, g_total=10_000, g_model=1000, g_runtime=500, g_safety=500)
    cap = oracle.cap(cfg)
    assert cap == 8000
    tm = 1000
    lo, hi = math.floor(0.5 * tm), math.floor(1.5 * tm)
    prev = None
    for A in range(0, 9000, 250):
        B = oracle.budget(cfg, tm, A, 300)
        assert lo <= B <= hi
        if prev is not None:
            assert B <= prev           # nonincreasing in active KV
        prev = B
    # gamma = 0: paused memory contributes nothing
    c0 = dict(cfg, gamma_num=0, gamma_den=1)
    assert oracle.budget(c0, tm, 7000, 900) == max(lo, min(hi, 8000 - 7000 - 900))
    c_wide = dict(cfg, beta_low=0.0, beta_high=100.0)
    assert oracle.budget(c_wide, 1000, 7000, 900) == 1000   # free 100 + paused 900
    c_half = dict(c_wide, gamma_num=1, gamma_den=2)
    assert oracle.budget(c_half, 1000, 7000, 901) == 99 + 450  # floor(901/2)
    # over-commitment: free floored at 0
    assert oracle.budget(c_wide, 1000, 8500, 0) == 0


def test_cap_7b_preset():
    """cap = floor((24 GiB - 12.1e9 - 1 GiB - 512 MiB)/458752) = 26286."""
    import tracegen
    assert oracle.cap(tracegen.PRESET_7B) == 26286


def test_hist_bins():
    assert [oracle.hist_bin(v) for v in range(16)] == list(range(16))
    assert oracle.hist_bin(16) == 16 and oracle.hist_bin(20) == 17 and oracle.hist_bin(31) == 19
    assert oracle.hist_bin(32) == 20
    b = [oracle.hist_bin(v) for v in range(0, 5000)]
    assert all(x <= y for x, y in zip(b, b[1:]))
    assert oracle.hist_bin(2**62) == 159


# ---- random scheduling (reading B8) ------------------------------
def test_splitmix64_known_answers():
    """The counter-based generator is SplitMix64's output function: its first
    outputs from state 0 and 1 are the published reference values."""
    assert oracle.splitmix64_mix(0) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64_mix(1) == 0x910A2DEC89025CC1


def test_random_ranking_reshuffles_every_iteration():
    """Random scheduling 'shuffles the request order': for a fixed
    pair of requests the relative order flips about half of the iterations,
    keys are spread uniformly, and different seeds give different orders."""
    import numpy as np
    flips = sum(oracle.random_key(7, 3, t) < oracle.random_key(7, 11, t) for t in range(4000))
    assert 1800 < flips < 2200
    keys = np.array([oracle.random_key(1, i, 99) for i in range(20000)], np.uint64)
    hist = np.bincount((keys >> np.uint64(28)).astype(np.int64), minlength=16)
    assert hist.min() > 20000 / 16 * 0.85 and hist.max() < 20000 / 16 * 1.15
    a = [oracle.random_key(1, i, 5) for i in range(64)]
    b = [oracle.random_key(2, i, 5) for i in range(64)]
    assert np.argsort(a).tolist() != np.argsort(b).tolist()
