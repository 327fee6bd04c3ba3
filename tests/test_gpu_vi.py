"""GPU parity of the single-instance full step's incremental order for value
(R3) and FCFS keys (step.cu, ti_incremental with vi): the previous order
minus the changed slots is merged with the changed ones after checking that
this step's words of the unchanged slots, taken in the previous order, still
increase; otherwise the step sorts.  Aimed at that check: a stream where
fp32 rounding re-orders waiting requests between steps (so the fallback
runs, which the oracle's own outputs confirm), random event streams with
prefix steps and bursts in between, and the cfg4 queue of 1M requests over
several steps.  Order, keys, grants, tier offsets and slot state must equal
the oracle's."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402
from test_gpu_step import random_events, compare, compare_slots  # noqa: E402


def _words(o):
    """(tier, key, slot) of every queued slot after an oracle step, as one
    orderable integer per slot (-1: not queued)."""
    n = int(o["n_active"][0])
    order = o["order"][0, :n].astype(np.int64)
    to = o["tier_off"][0]
    tier = np.zeros(n, np.int64)
    tier[to[1]:to[2]] = 1
    tier[to[2]:] = 2
    w = np.full(int(o["order"].shape[1]), -1, np.int64)
    w[order] = (tier << 62) | (o["keys"][0, :n].astype(np.int64) << 30) | order
    return w


@pytest.mark.parametrize("ranking", [0, 1])
def test_reordering_by_rounding(ranking):
    """Identical requests, one per step, in descending slot ids: equal values,
    so a waiting request's score is V - alpha*T*(t - arrival); with alpha*T
    far below fp32's spacing at V the keys tie in groups whose bounds move
    every step, and ties break by slot (here against the arrival order), so
    the previous order's unchanged words are often out of order."""
    MA = 400
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 10**6, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=ranking, budget_mode=1, l_static=30, alpha=1e-5)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, 1, MA)
    prev, out_of_order = None, 0
    for t in range(220):
        rec = oracle.records(1, kind=oracle.K_NEW, id=[MA - 1 - t], la=[100], lb=[10], ta=[0.0], flags=[0])
        assert st.enqueue(0, rec) == 0
        s.enqueue(0, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t))
        compare(g, o, 1, f"rounding rk{ranking} step {t}")
        w = _words(o)
        if prev is not None:
            po, pn, pa, pg = prev
            changed = np.zeros(MA, bool)
            changed[po[:pa][pg[:pa] > 0]] = True
            changed[MA - 1 - t] = True
            seq = w[po[:pn]][~changed[po[:pn]]]
            out_of_order += int(np.any(np.diff(seq) <= 0))
        n, a = int(o["n_active"][0]), int(o["admitted"][0])
        prev = (o["order"][0].astype(np.int64).copy(), n, a, o["grant"][0].copy())
    compare_slots(s, st, 1, f"rounding rk{ranking}")
    s.close()
    st.close()
    if ranking == 0:
        assert out_of_order > 20, out_of_order   # the fallback ran on many steps
    else:
        assert out_of_order == 0                 # FCFS keys never move


@pytest.mark.parametrize("seed,cap,pattern,ranking", [(5, 10**6, "full", 0), (6, 600, "mixed", 0),
                                                      (7, 10**6, "burst", 0), (8, 800, "full", 1)])
def test_vi_event_stream(seed, cap, pattern, ranking):
    """One instance, random events for 30 steps; 'mixed' puts prefix steps in
    between, 'burst' changes more slots than one merge takes."""
    rng = np.random.default_rng(seed)
    MA = 12_000 if pattern == "burst" else 3000
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=ranking, budget_mode=0, target_max=300,
                              alpha=1.5)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, 1, MA)
    for t in range(30):
        p_new = 0.8 if t == 0 else (0.9 if pattern == "burst" and t % 10 == 5 else 0.03)
        rec = random_events(rng, st.slots(0), t, p_new=p_new)
        if rec is not None:
            assert st.enqueue(0, rec) == 0
            s.enqueue(0, rec)
        o = st.step(t)
        assert o["rc"] == 0
        pre = pattern == "mixed" and t % 7 == 3
        g = s.step_result(s.step(t, prefix=pre))
        compare(g, o, 1, f"vi {pattern} step {t}", prefix=pre)
        if t % 5 == 4:
            compare_slots(s, st, 1, f"vi {pattern} step {t}")
    s.close()
    st.close()


def test_vi_cfg4_one_million_six_steps():
    """bench.py's cfg4 queue (1M requests, value ranking): the first step
    sorts, the next five merge."""
    n = 1_000_000
    rec = tracegen.cfg4_records(n)
    cfg, ip = tracegen.PRESET_CFG4, tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    for k in range(6):
        o = st.step(65536 + k)
        assert o["rc"] == 0
        g = s.step_result(s.step(65536 + k))
        compare(g, o, 1, f"cfg4 vi step {k}")
    assert np.array_equal(s.slots(0), st.slots(0))
    s.close()
    st.close()
