"""GPU parity of augsched_step (record intake, keys, device-wide LSD radix
sort, admission, resolution, grant accounting) against the oracle's step
mode: token limits, queue sizes, the full order, every key and every grant
must be identical, step after step."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402


def compare(g, o, n_inst, label, prefix=False):
    """Step outputs equal the oracle's: limits, queue sizes, admitted counts,
    and the order / keys / grants (the admitted prefix only when prefix)."""
    assert np.array_equal(g["B"], o["B"]), f"{label}: budget {g['B'][:4]} vs {o['B'][:4]}"
    assert np.array_equal(g["n_active"], o["n_active"]), f"{label}: n_active"
    assert np.array_equal(g["admitted"], o["admitted"]), f"{label}: admitted {g['admitted']} vs {o['admitted']}"
    for i in range(n_inst):
        n, a = int(o["n_active"][i]), int(o["admitted"][i])
        if prefix:
            n = a
        assert np.array_equal(g["order"][i, :n], o["order"][i, :n]), f"{label}: order inst {i}"
        assert np.array_equal(g["keys"][i, :n], o["keys"][i, :n]), f"{label}: keys inst {i}"
        assert np.array_equal(g["grant"][i, :a], o["grant"][i, :a]), f"{label}: grant inst {i}"
        if not prefix:
            # the full step writes zero grants beyond the admitted prefix
            assert not g["grant"][i, a:n].any(), f"{label}: stale grant beyond the prefix, inst {i}"
            assert np.array_equal(g["tier_off"][i], o["tier_off"][i]), f"{label}: tier offsets inst {i}"


def compare_slots(s, st, n_inst, label):
    """GPU slot state (augsched_step_export) and ledger equal the oracle's."""
    for i in range(n_inst):
        gs, os_ = s.slots(i), st.slots(i)
        assert np.array_equal(gs, os_), f"{label}: slot state inst {i}: rows " \
            f"{np.nonzero((gs != os_).any(1))[0][:8]}"
        assert s.ledger(i) == st.ledger(i), f"{label}: ledger inst {i}"


def test_G3_gpu():
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 10**6, g_model=1000)
    for rk in (0, 1):
        ip = tracegen.inst_params(1, base=tracegen.INST_G0, l_static=100, ranking=rk)
        rec = oracle.records(4, kind=oracle.K_NEW, id=[0, 1, 2, 3], la=[100, 20, 100, 20],
                             lb=[10, 10, 10, 10], ta=[0.0, 0.0, 2.0, 0.0], flags=[0, 0, 1, 1])
        st = oracle.Step(cfg, ip, 4)
        st.enqueue(0, rec)
        o = st.step(0)
        s = aug.Scheduler(cfg, ip, 1, 4)
        s.enqueue(0, rec)
        g = s.step_result(s.step(0))
        s.close()
        compare(g, o, 1, f"G3 ranking {rk}")
        want = [1, 3, 0, 2] if rk == 0 else [0, 1, 2, 3]
        assert list(g["order"][0]) == want


def random_events(rng, slots, now, p_new=0.3):
    """Valid engine events for one instance given its slot states."""
    recs = []
    for j, (stv, pol, ctx, kv, cpu, pend) in enumerate(slots):
        u = rng.random()
        if stv == 0 and u < p_new:
            recs.append(dict(kind=oracle.K_NEW, id=j, la=int(rng.integers(1, 300)),
                             lb=int(rng.integers(1, 80)), ta=float(rng.choice([0.0, 0.05, 1.0, 8.0])),
                             flags=int(rng.integers(0, 2))))
        elif stv == 1 and cpu == 0 and kv == ctx and pend == 0 and u < 0.3:
            if rng.random() < 0.6:
                recs.append(dict(kind=oracle.K_CALL, id=j, ta=float(rng.choice([0.0, 0.2, 3.0]))))
            else:
                recs.append(dict(kind=oracle.K_FINISH, id=j))
        elif stv == 4 and u < 0.35:
            recs.append(dict(kind=oracle.K_RETURN, id=j, la=int(rng.integers(1, 120)),
                             lb=int(rng.integers(1, 60)), ta=float(rng.choice([0.0, 0.5, 4.0])),
                             flags=int(rng.integers(0, 2))))
        elif stv in (2, 3) and u < 0.02:
            recs.append(dict(kind=oracle.K_FINISH, id=j))
    if not recs:
        return None
    cols = {k: [r.get(k, 0) for r in recs] for k in oracle.REC_FIELDS}
    return oracle.records(len(recs), **cols)


@pytest.mark.parametrize("seed,cap", [(1, 10**6), (2, 900), (3, 400)])
def test_random_event_stream(seed, cap):
    """4 instances x 64 slots (value, FCFS and random ranking), 40 steps of random NEW/CALL/RETURN/FINISH
    events; small caps force demotion and tail eviction every few steps."""
    rng = np.random.default_rng(seed)
    n_inst, MA = 4, 64
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=[0, 1, 0, 2], budget_mode=[1, 0, 0, 0],
                              l_static=150, target_max=[50, 200, 120, 90], alpha=[0.0, 0.0, 3.0, 0.0],
                              policy_mode=[0, 0, 0, 0], rank_seed=[0, 0, 0, 12345 + seed])
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(40):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t)
            if rec is not None:
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t))
        compare(g, o, n_inst, f"seed {seed} step {t}")
        compare_slots(s, st, n_inst, f"seed {seed} step {t}")
    s.close()


def test_state_violation_is_reported():
    cfg = dict(tracegen.PRESET_G0)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0)
    s = aug.Scheduler(cfg, ip, 1, 8)
    s.enqueue(0, oracle.records(1, kind=oracle.K_RETURN, id=[3], la=[5], lb=[5]))  # slot 3 not paused
    s.step(0)
    with pytest.raises(aug.AugschedError) as e:
        s.sync()
    assert e.value.code == aug.E_STATE
    s.close()


def test_cfg4_one_million_queue():
    """Config 4: one queue of 1,000,000 requests (512 running, 512 swapped,
    waiting 80% Stage I / 20% Stage II), 3 consecutive steps, full order."""
    n = 1_000_000
    rec = tracegen.cfg4_records(n)
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    t0 = 65536
    for k in range(3):
        o = st.step(t0 + k)
        g = s.step_result(s.step(t0 + k))
        compare(g, o, 1, f"cfg4 step {k}")
        assert int(g["B"][0]) == 750 and int(g["n_active"][0]) == n - 16
    s.close()


@pytest.mark.parametrize("seed,cap,ranking", [(11, 10**6, 0), (12, 700, 0), (13, 350, 2), (14, 500, 1)])
def test_prefix_step_event_stream(seed, cap, ranking):
    """augsched_step_prefix on one instance (256 slots) over 60 steps of
    random engine events: the admitted prefix, grants, limits and the slot
    state after every step equal the oracle's full-order step; small caps
    force the demotion / tail-eviction path."""
    rng = np.random.default_rng(seed)
    MA = 256
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=ranking, budget_mode=0, target_max=100,
                              alpha=1.5, rank_seed=seed)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, 1, MA)
    for t in range(60):
        rec = random_events(rng, st.slots(0), t, p_new=0.4)
        if rec is not None:
            assert st.enqueue(0, rec) == 0
            s.enqueue(0, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t, prefix=True))
        compare(g, o, 1, f"prefix seed {seed} step {t}", prefix=True)
        compare_slots(s, st, 1, f"prefix seed {seed} step {t}")
    s.close()


@pytest.mark.parametrize("seed,cap,ranking", [(31, 10**6, 0), (32, 500, 0), (33, 10**6, 1), (34, 500, 2)])
def test_prefix_step_anchor_event_stream(seed, cap, ranking):
    """A single-instance queue larger than the candidate capacity (12,000
    slots > 8,192): the first step takes the histogram fallback, later steps
    the speculative pass against the previous step's anchor slot; random
    NEW/CALL/RETURN/FINISH events move entries across the anchor and small
    caps force demotion and tail eviction; random ranking (a fresh shuffle
    every step, so no anchor) takes the histogram path on every step.  Every
    step equals the oracle's full-order step on the admitted prefix."""
    rng = np.random.default_rng(seed)
    MA = 12_000
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=ranking, budget_mode=0, target_max=300,
                              alpha=1.5, rank_seed=seed)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, 1, MA)
    for t in range(24):
        rec = random_events(rng, st.slots(0), t, p_new=0.85 if t == 0 else 0.05)
        if rec is not None:
            assert st.enqueue(0, rec) == 0
            s.enqueue(0, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t, prefix=True))
        compare(g, o, 1, f"anchor seed {seed} step {t}", prefix=True)
        assert int(o["n_active"][0]) > 8192 or t > 0
    s.close()


def test_prefix_and_full_steps_interleaved():
    """One single-instance handle (10,000 slots) alternating augsched_step
    and augsched_step_prefix: the prefix kernel keeps its counters clear
    across calls (epoch-tagged flags, no per-step memset) and the full step
    in between leaves nothing behind; every step equals the oracle's."""
    rng = np.random.default_rng(41)
    MA = 10_000
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 600, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=0, budget_mode=0, target_max=300, alpha=1.5)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, 1, MA)
    for t in range(16):
        rec = random_events(rng, st.slots(0), t, p_new=0.9 if t == 0 else 0.05)
        if rec is not None:
            assert st.enqueue(0, rec) == 0
            s.enqueue(0, rec)
        o = st.step(t)
        pre = t % 4 != 2
        g = s.step_result(s.step(t, prefix=pre))
        compare(g, o, 1, f"interleaved step {t} prefix={pre}", prefix=pre)
    s.close()


def test_prefix_step_cfg4_one_million_queue():
    """Config 4 through augsched_step_prefix: 6 consecutive steps over the
    1,000,000-request queue (the first through the histogram fallback, the
    rest through the anchored speculative pass); the admitted prefix equals
    the oracle's order."""
    n = 1_000_000
    rec = tracegen.cfg4_records(n)
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    t0 = 65536
    for k in range(6):
        o = st.step(t0 + k)
        g = s.step_result(s.step(t0 + k, prefix=True))
        compare(g, o, 1, f"cfg4 prefix step {k}", prefix=True)
        assert int(g["admitted"][0]) > 0
    s.close()


@pytest.mark.parametrize("n_inst,l_static", [(1, 20_000), (2, 150), (3, 9000)])
def test_prefix_step_falls_back_to_full_order(n_inst, l_static):
    """Handles the prefix selection does not cover (a limit above 8,192, or
    several instances) run the full step; the admitted prefix still equals
    the oracle's."""
    rng = np.random.default_rng(7)
    MA = 128
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 10**6, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, budget_mode=1, l_static=l_static)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(20):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=0.5)
            if rec is not None:
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(t)
        g = s.step_result(s.step(t, prefix=True))
        compare(g, o, n_inst, f"fallback step {t}", prefix=True)
    s.close()


@pytest.mark.parametrize("seed,cap", [(21, 10**6), (22, 900), (23, 400)])
def test_prefix_step_multi_instance_event_stream(seed, cap):
    """augsched_step_prefix on a 4-instance handle (one CTA per instance:
    keys in shared memory, count-weighted radix select, sort, admission,
    resolution, apply): 40 steps of random events, value / FCFS / random
    ranking, small caps forcing demotion and tail eviction."""
    rng = np.random.default_rng(seed)
    n_inst, MA = 4, 64
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=[0, 1, 0, 2], budget_mode=[1, 0, 0, 0],
                              l_static=150, target_max=[50, 200, 120, 90], alpha=[0.0, 0.0, 3.0, 0.0],
                              rank_seed=[0, 0, 0, 99 + seed])
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(40):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t)
            if rec is not None:
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t, prefix=True))
        compare(g, o, n_inst, f"multi prefix seed {seed} step {t}", prefix=True)
        compare_slots(s, st, n_inst, f"multi prefix seed {seed} step {t}")
    s.close()


# ------------------------------------------------------------------ round-2 boundary checks
def _g0(cap=10**6):
    return dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)


def _imp(rows):
    n = len(rows)
    col = lambda k, d=0: [r.get(k, d) for r in rows]
    return oracle.records(n, kind=col("kind", oracle.K_IMPORT), id=col("id"), la=col("la", 1), lb=col("lb", 1),
                          flags=[(r.get("st", 3) << 4) | (r.get("pol", 2) << 8) for r in rows],
                          last=col("last"), ctx=col("ctx"), kv=col("kv"), cpu=col("cpu"), pend=col("pend"))


@pytest.mark.parametrize("prefix", [False, True])
def test_r2_golden_pins_on_gpu(prefix):
    """The hand-worked step-mode goldens P3 (demotion order) and P4
    (eviction of a slot mid swap-in; admitted = prefix length with a
    cancelled grant inside it) of tests/golden/r2_pins.json, on the GPU."""
    import json
    import os
    G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "r2_pins.json")))
    g3 = G["P3_demotion_order_step"]
    s = aug.Scheduler(_g0(61), tracegen.inst_params(1, base=tracegen.INST_G0, l_static=100), 1, 5)
    s.enqueue(0, _imp([dict(id=0, st=4, pol=0, ctx=15, kv=15), dict(id=1, st=4, pol=0, ctx=5, kv=5),
                       dict(id=2, st=4, pol=0, ctx=15, kv=15), dict(id=3, st=1, ctx=10, kv=10, la=1, lb=1),
                       dict(id=4, st=3, pend=25, la=25, lb=1)]))
    g = s.step_result(s.step(10, prefix=prefix))
    assert int(g["admitted"][0]) == g3["admitted"] and int(g["n_active"][0]) == g3["n_active"]
    assert g["order"][0][:2].tolist() == g3["order"] and g["grant"][0][:2].tolist() == g3["grant"]
    assert s.slots(0).tolist() == g3["slots_after"]
    assert s.ledger(0) == (g3["ledger_after"]["A"], g3["ledger_after"]["P"])
    s.close()
    g4 = G["P4_evict_mid_swapin_step"]
    s = aug.Scheduler(_g0(55), tracegen.inst_params(1, base=tracegen.INST_G0, l_static=100), 1, 2)
    s.enqueue(0, _imp([dict(id=0, st=1, ctx=10, kv=10, la=1, lb=1),
                       dict(id=1, st=1, ctx=100, kv=40, cpu=60, la=2, lb=2)]))
    for now, key in ((10, "step1"), (11, "step2")):
        g = s.step_result(s.step(now, prefix=prefix))
        w = g4[key]
        assert int(g["admitted"][0]) == w["admitted"]
        assert g["order"][0].tolist() == w["order"] and g["grant"][0].tolist() == w["grant"]
        assert s.slots(0).tolist() == w["slots_after"]
        assert s.ledger(0) == (w["ledger_after"]["A"], w["ledger_after"]["P"])
    s.close()


def test_stale_grants_cleared_by_full_step():
    """a full step after a step with a longer admitted prefix
    writes zeros (not the old grants) at the positions beyond its own prefix."""
    cfg = _g0()
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, l_static=100)
    for pre0 in (True, False):
        st = oracle.Step(cfg, ip, 16)
        s = aug.Scheduler(cfg, ip, 1, 16)
        rec = _imp([dict(id=j, st=3, pend=5, la=5, lb=1) for j in range(8)])
        st.enqueue(0, rec)
        s.enqueue(0, rec)
        o = st.step(0)
        g = s.step_result(s.step(0, prefix=pre0))
        compare(g, o, 1, "stale t0", prefix=pre0)
        assert int(g["admitted"][0]) == 8
        rec = oracle.records(12, kind=[oracle.K_FINISH] * 6 + [oracle.K_NEW] * 6, id=list(range(6)) + list(range(8, 14)),
                             la=[0] * 6 + [200] * 6, lb=[0] * 6 + [1] * 6)
        st.enqueue(0, rec)
        s.enqueue(0, rec)
        o = st.step(1)
        g = s.step_result(s.step(1))
        assert int(o["admitted"][0]) == 3 and int(o["n_active"][0]) == 8
        compare(g, o, 1, "stale t1")
        s.close()


def test_duplicate_slot_records_are_state_violations():
    """two records for one slot in the same record phase (CALL +
    FINISH, two FINISHes, two NEWs, RETURN + NEW) are state violations: the
    first in the oracle's processing order applies, the others are rejected
    with E_STATE, and every slot's state equals the oracle's."""
    cfg = _g0()
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, l_static=1000)
    st = oracle.Step(cfg, ip, 8)
    s = aug.Scheduler(cfg, ip, 1, 8)
    init = _imp([dict(id=0, st=1, ctx=10, kv=10), dict(id=1, st=1, ctx=12, kv=12),
                 dict(id=2, st=4, pol=2, ctx=20), dict(id=3, st=3, pend=4, la=4)])
    st.enqueue(0, init)
    s.enqueue(0, init)
    st.step(0)
    s.step_result(s.step(0))
    K = oracle
    dup = oracle.records(7, kind=[K.K_CALL, K.K_FINISH, K.K_FINISH, K.K_FINISH, K.K_NEW, K.K_NEW, K.K_RETURN],
                         id=[0, 0, 1, 1, 5, 5, 2], la=[0, 0, 0, 0, 7, 9, 3], lb=[0, 0, 0, 0, 2, 2, 1],
                         ta=[0.0, 0, 0, 0, 0, 0, 0])
    # RETURN + NEW on slot 2 (paused): the return applies, the NEW is rejected
    dup2 = oracle.records(1, kind=[K.K_NEW], id=[2], la=[5], lb=[1])
    for r in (dup, dup2):
        st.enqueue(0, r)
        s.enqueue(0, r)
    o = st.step(1)
    assert o["rc"] == -4
    s.step(1)
    with pytest.raises(aug.AugschedError) as e:
        s.sync()
    assert e.value.code == aug.E_STATE
    assert np.array_equal(s.slots(0), st.slots(0))
    assert s.ledger(0) == st.ledger(0)
    s.close()


def test_import_last_in_the_future_is_rejected():
    cfg = _g0()
    ip = tracegen.inst_params(1, base=tracegen.INST_G0)
    st = oracle.Step(cfg, ip, 4)
    s = aug.Scheduler(cfg, ip, 1, 4)
    rec = _imp([dict(id=0, st=3, pend=5, last=7), dict(id=1, st=3, pend=5, last=3)])
    st.enqueue(0, rec)
    s.enqueue(0, rec)
    assert st.step(5)["rc"] == -4
    s.step(5)
    with pytest.raises(aug.AugschedError) as e:
        s.sync()
    assert e.value.code == aug.E_STATE
    assert np.array_equal(s.slots(0), st.slots(0))
    s.close()


def test_now_must_fit_u32_and_not_run_backwards():
    s = aug.Scheduler(_g0(), tracegen.inst_params(1, base=tracegen.INST_G0), 1, 4)
    with pytest.raises(aug.AugschedError) as e:
        s.step(2**32)
    assert e.value.code == aug.E_INVALID
    s.step(10)
    with pytest.raises(aug.AugschedError) as e:
        s.step(9, prefix=True)
    assert e.value.code == aug.E_INVALID
    s.step(10)        # equal is fine
    s.sync()
    s.close()


@pytest.mark.parametrize("n_inst,MA,cap", [(3, 100, 10**6), (2, 3000, 900), (2, 5000, 10**6), (5, 1500, 600)])
def test_batched_full_order_shapes(n_inst, MA, cap):
    """The batched full-order kernel (one CTA per instance, shared-memory LSD
    sort) at slot counts that are not powers of two and at its 512-thread
    size (MA > 4,096): 12 steps of random events, every output and the slot
    state equal the oracle's."""
    rng = np.random.default_rng(MA + n_inst)
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(n_inst, base=tracegen.INST_G0, ranking=[0, 1, 0, 2, 0][:n_inst],
                              budget_mode=0, target_max=[300, 200, 120, 90, 400][:n_inst],
                              alpha=[1.5, 0.0, 3.0, 0.0, 0.2][:n_inst], rank_seed=7)
    st = oracle.Step(cfg, ip, MA)
    s = aug.Scheduler(cfg, ip, n_inst, MA)
    for t in range(12):
        for i in range(n_inst):
            rec = random_events(rng, st.slots(i), t, p_new=0.7 if t == 0 else 0.1)
            if rec is not None:
                assert st.enqueue(i, rec) == 0
                s.enqueue(i, rec)
        o = st.step(t)
        assert o["rc"] == 0
        g = s.step_result(s.step(t))
        compare(g, o, n_inst, f"batched MA={MA} step {t}")
        compare_slots(s, st, n_inst, f"batched MA={MA} step {t}")
    s.close()
