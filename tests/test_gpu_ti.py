"""GPU parity of ranking mode 3 (reading B12: the
time-invariant key V + alpha*last*T) against the oracle: the simulator, the
batched step, and the single-instance full step whose order is kept
incrementally (the slots changed since the last step are merged into the
previous order), including the fallbacks (first step, more changed slots
than one merge takes, a prefix step in between)."""
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


def test_simulate_mode3_equals_oracle():
    tr = tracegen.gen_traces(4, 800, [2.0, 4.0, 6.0, 8.0], seed=31)
    n = 16
    ip = tracegen.inst_params(n, ranking=3, alpha=np.array([0.0, 4.6e6, 4.6e7, 4.6e8] * 4),
                              target_max=np.repeat([250, 500, 750, 1000], 4))
    tid = (np.arange(n) % 4).astype(np.uint32)
    s = aug.Scheduler(tracegen.PRESET_7B, ip, n, 800)
    g = s.simulate_host(tr, tid)
    s.close()
    o = oracle.simulate(tracegen.PRESET_7B, ip, tr, tid)
    assert g.tobytes() == o.tobytes()


@pytest.mark.parametrize("seed,cap,pattern", [(1, 10**6, "full"), (2, 700, "full"), (3, 500, "mixed"),
                                              (4, 10**6, "burst")])
def test_incremental_full_step_stream(seed, cap, pattern):
    """One instance, 3,000 slots, 30 steps of random events in mode 3; 'mixed'
    puts prefix steps in between (the next full step sorts again), 'burst'
    creates more changed slots than one merge takes at some steps."""
    rng = np.random.default_rng(seed)
    MA = 12_000 if pattern == "burst" else 3000
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=3, budget_mode=0, target_max=300, alpha=1.5)
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
        compare(g, o, 1, f"ti {pattern} step {t}", prefix=pre)
        if t % 5 == 4:
            compare_slots(s, st, 1, f"ti {pattern} step {t}")
    s.close()


def test_incremental_full_step_cfg4_one_million():
    """Config 4 in mode 3: six consecutive full-order steps over the 1M queue
    (the first sorts, the next five merge ~1,000 changed slots each)."""
    n = 1_000_000
    rec = tracegen.cfg4_records(n)
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(1, ranking=3)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    t0 = 65536
    for k in range(6):
        o = st.step(t0 + k)
        g = s.step_result(s.step(t0 + k))
        compare(g, o, 1, f"cfg4 ti step {k}")
    assert np.array_equal(s.slots(0), st.slots(0))
    s.close()


def test_batched_mode3_stream():
    rng = np.random.default_rng(9)
    n_inst, MA = 4, 256
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 600, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=3, budget_mode=0, target_max=120,
                              alpha=[0.0, 1.0, 5.0, 50.0])
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(20):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=0.6 if t == 0 else 0.1)
            if rec is not None:
                st.enqueue(i, rec)
                s.enqueue(i, rec)
        o = st.step(t)
        for pre in (False,):
            g = s.step_result(s.step(t, prefix=pre))
            compare(g, o, n_inst, f"batched ti step {t}", prefix=pre)
        compare_slots(s, st, n_inst, f"batched ti step {t}")
    s.close()


def test_incremental_edge_cases():
    """Mode 3 with alpha = 0 (the order equals R3's), a static limit of 0
    (nothing admitted, so no grant changes a word), and a queue that empties
    (every slot finishes) and refills."""
    rng = np.random.default_rng(77)
    MA = 500
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 10**6, g_model=1000)
    for kw in (dict(alpha=0.0, budget_mode=0), dict(alpha=2.0, budget_mode=1, l_static=0)):
        ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=3, target_max=100, **kw)
        st = oracle.Step(cfg, ip, MA)
        s = aug.Scheduler(cfg, ip, 1, MA)
        for t in range(16):
            if t == 8:   # finish every queued request, then new arrivals
                sl = st.slots(0)
                ids = [j for j in range(MA) if sl[j][0] in (1, 2, 3)]
                rec = oracle.records(len(ids), kind=oracle.K_FINISH, id=ids) if ids else None
            else:
                rec = random_events(rng, st.slots(0), t, p_new=0.5 if t in (0, 9) else 0.05)
            if rec is not None:
                st.enqueue(0, rec)
                s.enqueue(0, rec)
            o = st.step(t)
            compare(s.step_result(s.step(t)), o, 1, f"ti edge {kw} step {t}")
        compare_slots(s, st, 1, "ti edge")
        s.close()
