"""Round-2 pins of oracle paths the G1-G8 schedules leave open
(tests/golden/r2_pins.json, each case hand-worked from the cited passage):

- P1/P2: C_other of Eq.5 at call issuance excludes the caller's own KV
  (R7, R13), in the simulator and in step mode;
- P3: R20 demotion order (kv desc, id asc) in step mode;
- P4: R20 tail eviction of a request that was mid swap-in drops its CPU copy
  too (reading B2), and `admitted` is the admission-prefix length
  (Algorithm 1), so an eviction can leave a zero grant inside it;
- P5: a NEW -> CALL -> RETURN -> FINISH record stream (G5 in step mode);
- P6: the 5x-relaxed SLO differs from the 1x one;
- Proposition 1 in exact integers, exhaustively, and the
  simulator's service time against Eq.(Tt-basic).

`tools/oracle_mutants.py` checks that each plausible mutation of these paths
fails at least one test here."""
import itertools
import json
import os
import struct

import numpy as np
import pytest

import oracle
import tracegen
from oracle import K_CALL, K_FINISH, K_IMPORT, K_NEW, K_RETURN

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "r2_pins.json")))
T = 100_000
ST_RUN, ST_SWAP, ST_WAIT, ST_PAUSED = 1, 2, 3, 4
P_, S_, D_ = 0, 1, 2


def cfg0(cap=1_000_000, **kw):
    return dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000, **kw)


def inst0(B, **kw):
    return tracegen.inst_params(1, base=tracegen.INST_G0, l_static=B, **kw)


def req(arr, l_pre, segs):
    out = []
    for s in segs:
        out.append((s[0], s[0], 0, 0.0, 0) if len(s) == 1 else (s[0], s[0], s[1], s[2], s[3]))
    return {"arr": arr, "l_pre": l_pre, "segs": out}


def imp(slots):
    """IMPORT records from dicts {id, st, pol, la, lb, ctx, kv, cpu, pend} (stage I features)."""
    n = len(slots)
    col = lambda k, d=0: [s.get(k, d) for s in slots]
    flags = [(s["st"] << 4) | (s.get("pol", D_) << 8) for s in slots]
    return oracle.records(n, kind=K_IMPORT, id=col("id"), la=col("la", 1), lb=col("lb", 1),
                          flags=flags, last=col("last", 0), ctx=col("ctx"), kv=col("kv"),
                          cpu=col("cpu"), pend=col("pend"))


def key_of(v):
    u = struct.unpack("<I", struct.pack("<f", v))[0]
    return (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)


# ------------------------------------------------------------------ P1 / P2
def test_P1_issuance_cother_excludes_own_kv_sim():
    g = G["P1_issuance_cother_sim"]
    reqs = [req(r["arr"], r["l_pre"], r["segs"]) for r in g["requests"]]
    tr = tracegen.from_requests([reqs])
    rec, ft, fin = oracle.simulate_detail(cfg0(s_out=1), inst0(100), tr)
    assert rec["err"] == 0
    assert rec["calls_discard"] == g["calls_discard"] and rec["calls_preserve"] == g["calls_preserve"]
    assert rec["calls_swap"] == g["calls_swap"]
    assert list(fin) == g["finish_iter"] and list(ft) == g["first_token_iter"]
    assert rec["busy_steps"] == g["busy_steps"] and rec["tokens_granted"] == g["tokens_granted"]
    assert rec["slo_ok"] == g["slo_ok"]


def test_P2_issuance_cother_excludes_own_kv_step():
    g = G["P2_issuance_cother_step"]
    st = oracle.Step(cfg0(s_out=1), inst0(100), max_active=2)
    st.enqueue(0, imp([dict(id=0, st=ST_RUN, ctx=10, kv=10), dict(id=1, st=ST_RUN, ctx=19, kv=19)]))
    o = st.step(5)
    assert o["rc"] == 0 and list(o["grant"][0]) == [1, 1]
    assert st.ledger(0) == (31, 0)
    st.enqueue(0, oracle.records(1, kind=K_CALL, id=0, ta=0.35))
    o = st.step(6)
    assert o["rc"] == 0
    want = g["slot0_after"]
    assert st.slots(0)[0].tolist() == [want[k] for k in ("status", "policy", "ctx", "kv", "cpu", "pend")]
    assert st.ledger(0) == (g["ledger_after"]["A"], g["ledger_after"]["P"])


# ------------------------------------------------------------------ P3 demotion order
def test_P3_demotion_kv_desc_id_asc_step():
    g = G["P3_demotion_order_step"]
    st = oracle.Step(cfg0(cap=61), inst0(100), max_active=5)
    st.enqueue(0, imp([
        dict(id=0, st=ST_PAUSED, pol=P_, ctx=15, kv=15),
        dict(id=1, st=ST_PAUSED, pol=P_, ctx=5, kv=5),
        dict(id=2, st=ST_PAUSED, pol=P_, ctx=15, kv=15),
        dict(id=3, st=ST_RUN, ctx=10, kv=10, la=1, lb=1),
        dict(id=4, st=ST_WAIT, pend=25, la=25, lb=1),
    ]))
    assert st.ledger(0) == (0, 0)          # records apply at the step
    o = st.step(10)
    assert o["rc"] == 0
    assert o["B"][0] == g["B"] and o["n_active"][0] == g["n_active"] and o["admitted"][0] == g["admitted"]
    n = int(o["n_active"][0])
    assert o["order"][0][:n].tolist() == g["order"] and o["grant"][0][:n].tolist() == g["grant"]
    assert st.slots(0).tolist() == g["slots_after"]
    assert st.ledger(0) == (g["ledger_after"]["A"], g["ledger_after"]["P"])


# ------------------------------------------------------------------ P4 eviction mid swap-in
def test_P4_eviction_drops_cpu_copy_and_admitted_is_prefix_length():
    g = G["P4_evict_mid_swapin_step"]
    st = oracle.Step(cfg0(cap=55), inst0(100), max_active=2)
    st.enqueue(0, imp([dict(id=0, st=ST_RUN, ctx=10, kv=10, la=1, lb=1),
                       dict(id=1, st=ST_RUN, ctx=100, kv=40, cpu=60, la=2, lb=2)]))
    for now, key in ((10, "step1"), (11, "step2")):
        o = st.step(now)
        w = g[key]
        assert o["rc"] == 0
        assert o["B"][0] == w["B"] and o["n_active"][0] == w["n_active"]
        assert o["admitted"][0] == w["admitted"]
        assert o["order"][0].tolist() == w["order"] and o["grant"][0].tolist() == w["grant"]
        assert st.slots(0).tolist() == w["slots_after"]
        assert st.ledger(0) == (w["ledger_after"]["A"], w["ledger_after"]["P"])
    # admitted counts a cancelled grant: prefix length 2, one grant > 0
    assert int((o["grant"][0] > 0).sum()) == 1 < o["admitted"][0]


# ------------------------------------------------------------------ P5 record stream
def test_P5_new_call_return_finish_stream():
    g = G["P5_step_stream"]
    st = oracle.Step(cfg0(), inst0(100), max_active=1)
    st.enqueue(0, oracle.records(1, kind=K_NEW, id=0, la=10, lb=2, ta=0.3, flags=1))
    events = {3: oracle.records(1, kind=K_CALL, id=0, ta=0.3),
              6: oracle.records(1, kind=K_RETURN, id=0, la=5, lb=1, ta=0.0, flags=0),
              9: oracle.records(1, kind=K_FINISH, id=0)}
    for now in (0, 1, 2, 3, 6, 7, 8, 9):
        if now in events:
            st.enqueue(0, events[now])
        o = st.step(now)
        assert o["rc"] == 0
        want = g["grants"][str(now)]
        if want is None:
            assert o["n_active"][0] == 0 and o["admitted"][0] == 0
        else:
            assert o["n_active"][0] == 1 and o["admitted"][0] == 1
            assert int(o["grant"][0][0]) == want
        if now == 0:
            assert int(o["keys"][0][0]) == key_of(g["values"]["V1"])
        if now == 6:
            assert int(o["keys"][0][0]) == key_of(g["values"]["V2"])
        if str(now) in g["A_after"]:
            assert st.ledger(0)[0] == g["A_after"][str(now)]
    s = st.slots(0)[0].tolist()
    assert s == [0, 2, 0, 0, 0, 0]     # slot empty again


def test_P5_call_swap_sets_cpu_copy():
    """R21: a Swap call moves the whole context to the CPU copy at issuance."""
    st = oracle.Step(cfg0(), inst0(100), max_active=1)
    st.enqueue(0, oracle.records(1, kind=K_NEW, id=0, la=10, lb=2, ta=0.3, flags=1))
    for now in (0, 1, 2):
        st.step(now)
    st.enqueue(0, oracle.records(1, kind=K_CALL, id=0, ta=0.3))
    st.step(3)
    assert st.slots(0)[0].tolist() == [ST_PAUSED, S_, 12, 0, 12, 0]
    assert st.ledger(0) == (0, 0)


# ------------------------------------------------------------------ P6 5x SLO
def test_P6_slo_5x_differs_from_1x():
    g = G["P6_slo_5x"]
    reqs = [req(0, 10, [(1, 5_000_000, 0.0, 2), (1,)]), req(300_000, 25, [(1,)])]
    tr = tracegen.from_requests([reqs])
    rec, ft, fin = oracle.simulate_detail(cfg0(30), inst0(30), tr)
    assert rec["slo_ok"] == g["slo_ok"] and rec["slo_ok_5x"] == g["slo_ok_5x"]


# ------------------------------------------------------------------ Proposition 1
def test_proposition1_exact_integers():
    """with T_t,i = I_t (G_i + A_i / N) and T_l,i = G_i + A_i,
    (T_l2 > T_l1 and T_t1 > T_t2)  <=>  (T_l2 > T_l1 and
    T_l2 - T_l1 < (1 - 1/N)(A_2 - A_1)), checked exhaustively with both sides
    multiplied by N (integers, no rounding)."""
    mism = 0
    for N in range(1, 9):
        for G1, A1, G2, A2 in itertools.product(range(7), repeat=4):
            Tl1, Tl2 = G1 + A1, G2 + A2
            Tt1, Tt2 = N * G1 + A1, N * G2 + A2          # N * T_t / I_t
            lhs = Tl2 > Tl1 and Tt1 > Tt2
            rhs = Tl2 > Tl1 and N * (Tl2 - Tl1) < (N - 1) * (A2 - A1)
            mism += lhs != rhs
    assert mism == 0


@pytest.mark.parametrize("G0,A,G1,B", [(3, 100, 2, 50), (1, 150, 4, 50), (5, 50, 1, 25), (2, 0, 3, 10)])
def test_service_time_matches_eq_Tt_basic(G0, A, G1, B):
    """Eq.(Tt-basic): a lone request with a zero-duration,
    Preserve call is served in G iterations of decode plus A/N of
    assimilation (A a multiple of the per-iteration limit B = N) -- here
    plus ceil(L/B) prefill iterations (R22) and no idle iteration."""
    L = 2 * B
    tr = tracegen.from_requests([[req(0, L, [(G0, 0, 0.0, A), (G1,)])]])
    rec, ft, fin = oracle.simulate_detail(cfg0(), inst0(B, policy_mode=1), tr)
    assert rec["calls_preserve"] == 1 and rec["completed"] == 1
    want = L // B + G0 + A // B + G1
    assert rec["busy_steps"] == want
    assert fin[0] == want           # no idle iteration: the call returns at the next boundary


def _run(key, cap, B, cfg_kw=None, **kw):
    g = G[key]
    reqs = [req(r["arr"], r["l_pre"], r["segs"]) for r in g["requests"]]
    tr = tracegen.from_requests([reqs])
    rec, ft, fin = oracle.simulate_detail(cfg0(cap, **(cfg_kw or {})), inst0(B, **kw), tr)
    assert rec["err"] == 0
    return g, rec, ft, fin


def test_P7_arrivals_use_snapshot_taken_before_returns():
    g, rec, ft, fin = _run("P7_snapshot_before_returns_sim", 1_000_000, 11, dict(s_out=1))
    assert list(ft) == g["first_token_iter"]


def test_P8_demotion_kv_desc_sim():
    g, rec, ft, fin = _run("P8_demotion_order_sim", 40, 100, dict(s_out=1))
    assert rec["demotions"] == g["demotions"] and rec["evictions"] == g["evictions"]
    assert list(fin) == g["finish_iter"] and rec["calls_preserve"] == g["calls_preserve"]


def test_P9_eviction_mid_swapin_recomputes_sim():
    g, rec, ft, fin = _run("P9_evict_mid_swapin_sim", 35, 100, dict(s_in=5), ranking=1)
    assert rec["evictions"] == g["evictions"] and list(fin) == g["finish_iter"]
    assert rec["busy_steps"] == g["busy_steps"] and rec["tokens_granted"] == g["tokens_granted"]
    assert rec["calls_swap"] == g["calls_swap"]


def test_P10_slo_5x_ttft_term():
    g, rec, ft, fin = _run("P10_slo5x_ttft", 1_000_000, 10, ranking=1)
    assert list(fin) == g["finish_iter"]
    assert rec["slo_ok"] == g["slo_ok"] and rec["slo_ok_5x"] == g["slo_ok_5x"]


def test_P11_last_scheduled_time_set_on_grant():
    g, rec, ft, fin = _run("P11_last_on_grant_sim", 1_000_000, 10, alpha=1000.0)
    assert list(ft) == g["first_token_iter"] and list(fin) == g["finish_iter"]


def test_R28_incomplete_counter():
    """R28 / S:481: a run stopped at the horizon counts the requests still
    unfinished.  G4's request (prefill at t0, tokens at t1..t5,
    finish at iteration 6): a run with max_iters 5 stops before its last
    decode (1 incomplete), max_iters 6 lets it finish (0)."""
    tr = tracegen.from_requests([[req(0, 10, [(5,)])]])
    for mi, inc in ((5, 1), (6, 0), (1, 1)):
        rec, ft, fin = oracle.simulate_detail(cfg0(), inst0(15), tr, max_iters=mi)
        assert rec["incomplete"] == inc and rec["completed"] == 1 - inc


def test_R28_completed_plus_incomplete_is_n():
    tr = tracegen.gen_traces(3, 150, [2.0, 4.0, 8.0], seed=5)
    for mi in (300, 2000, 2**40):
        res = oracle.simulate(tracegen.PRESET_7B, tracegen.inst_params(3), tr, np.arange(3, dtype=np.uint32),
                              max_iters=mi)
        for x in res:
            d = oracle.as_dict(x)
            assert d["completed"] + d["incomplete"] == d["n_requests"]
