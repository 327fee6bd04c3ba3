"""GPU parity of the batched full step's incremental order (step.cu,
full_multi_kernel): each instance's previous order minus the changed slots
and the out-of-place words is merged with the rest instead of re-sorted.
Aimed at what could make it part from the sorted-order definition of
Algorithm 1: fp32 ties that re-form from step to step (alpha 0,
identical requests), steps with no records at all (every waiting score moves
by the same alpha*T), bursts larger than the merge buffer (the full sort runs
instead), prefix steps in between (the kept order is dropped), FCFS, random
and time-invariant rankings in the same handle, and eviction under tight
memory.  Every output (limit, queue size, admitted count, order, keys,
grants, tier segments) and the slot state must equal the oracle's."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402
from test_gpu_step import compare, compare_slots, random_events  # noqa: E402


def _new_records(ids, la, lb, ta=0.0, flags=0):
    n = len(ids)
    return oracle.records(n, kind=oracle.K_NEW, id=list(ids), la=list(la), lb=list(lb), ta=[ta] * n,
                          flags=[flags] * n)


@pytest.mark.parametrize("seed,cap", [(21, 10**6), (22, 700)])
def test_incremental_event_stream(seed, cap):
    """8 instances x 300 slots, every ranking mode, 36 full steps of random
    events; identical prompts (equal values) so fp32 ties are common."""
    rng = np.random.default_rng(seed)
    n_inst, MA = 8, 300
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=[0, 1, 0, 3, 0, 2, 0, 3],
                              budget_mode=[0, 1, 0, 0, 1, 0, 0, 0], l_static=200,
                              target_max=[60, 200, 120, 90, 150, 80, 300, 40],
                              alpha=[0.0, 0.0, 3.0, 2.0, 1e-3, 0.0, 50.0, 0.0],
                              rank_seed=[0, 0, 0, 0, 0, 77 + seed, 0, 0])
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    # a block of identical requests per instance first (equal V: key ties)
    for i in range(n_inst):
        rec = _new_records(range(0, 120), [50] * 120, [10] * 120)
        assert st.enqueue(i, rec) == 0
        s.enqueue(i, rec)
    for t in range(36):
        if t % 5 != 4 and t > 0:   # every fifth step has no records: the pure time shift
            for i in range(n_inst):
                rec = random_events(rng, st.slots(i), t, p_new=0.1)
                if rec is not None:
                    assert st.enqueue(i, rec) == 0
                    s.enqueue(i, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t))
        compare(g, o, n_inst, f"seed {seed} step {t}")
        compare_slots(s, st, n_inst, f"seed {seed} step {t}")
    s.close()
    st.close()


def test_incremental_bursts_and_prefix_steps():
    """2 instances x 2,048 slots: a 2,048-request burst (beyond the merge
    buffer: full sort), quiet steps, a second burst of 600, and prefix steps
    interleaved (each drops the kept order)."""
    n_inst, MA = 2, 2048
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(n_inst, alpha=[4.6e7, 0.0], ranking=[0, 0])
    rng = np.random.default_rng(5)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    plan = {0: (0, 1400), 6: (1400, 2000)}
    pre = {3, 9}
    for t in range(14):
        if t in plan:
            a, b = plan[t]
            for i in range(n_inst):
                rec = _new_records(range(a, b), rng.integers(1, 400, b - a), rng.integers(1, 60, b - a))
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(65536 + t)
        assert o["rc"] == 0
        p = t in pre
        g = s.step_result(s.step(65536 + t, prefix=p))
        compare(g, o, n_inst, f"burst step {t} prefix={p}", prefix=p)
        compare_slots(s, st, n_inst, f"burst step {t}")
    s.close()
    st.close()


def test_bench_workload_many_steps():
    """bench.py step_multi's records on 256 instances, 12 consecutive full
    steps (the bench times steps after its warm-up: all incremental)."""
    n_inst, ma = 256, 2048
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(n_inst)
    rec = tracegen.cfg4_records(ma, n_running=16, n_swapped=16, n_paused=4)
    st = oracle.Step(cfg, ip, ma)
    s = aug.Scheduler(cfg, ip, n_inst, ma)
    for i in range(n_inst):
        assert st.enqueue(i, rec) == 0
        s.enqueue(i, rec)
    for k in range(12):
        o = st.step(65536 + k)
        assert o["rc"] == 0
        g = s.step_result(s.step(65536 + k))
        compare(g, o, n_inst, f"bench workload step {k}")
    for i in (0, 255):
        assert np.array_equal(s.slots(i), st.slots(i)), f"slots inst {i}"
    s.close()
    st.close()


@pytest.mark.parametrize("MA", [200, 1000, 4000, 8000])
def test_incremental_every_block_shape(MA):
    """Every template shape of the batched kernel (256 threads x 1, 4, 16
    words per thread; 512 x 16) over 12 steps with a burst of new requests
    and tight memory; FCFS, value and time-invariant rankings."""
    rng = np.random.default_rng(MA)
    n_inst = 3
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 4 * MA, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=[0, 1, 3], budget_mode=0,
                              target_max=[80, 160, 400], alpha=[2.0, 0.0, 0.5])
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(12):
        p_new = 0.6 if t in (0, 7) else 0.05
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=p_new)
            if rec is not None:
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t))
        compare(g, o, n_inst, f"MA {MA} step {t}")
    compare_slots(s, st, n_inst, f"MA {MA}")
    s.close()
    st.close()
