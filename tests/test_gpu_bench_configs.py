"""Parity at exactly the configurations bench.py times:

- augsched_step_prefix on one queue of 4,194,304 and of 16,000,000 requests
  (the size sweep; the phase loops take several trips per CTA), four steps:
  the first through the histogram fallback, the rest through the anchored
  speculative pass;
- the batched scheduler, 4,096 instances x 2,048 slots, through
  augsched_step (the per-instance shared-memory sort, two instance bytes in
  the device-wide fallback) and augsched_step_prefix (pf_sortE<256, 10>);
- config 5 (65,536 instances) advanced in the bench's 1,500-iteration
  windows through iteration 37,500 (5 warm-up + 20 timed windows), a sample
  of instances re-simulated by the oracle.

Every compared value comes from oracle/ on the same seeded inputs."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402


def check_step(g, o, n_inst, label, prefix):
    assert np.array_equal(g["B"], o["B"]), label
    assert np.array_equal(g["n_active"], o["n_active"]), label
    assert np.array_equal(g["admitted"], o["admitted"]), label
    if prefix:
        for i in range(n_inst):
            a = int(o["admitted"][i])
            assert np.array_equal(g["order"][i, :a], o["order"][i, :a]), f"{label}: order inst {i}"
            assert np.array_equal(g["keys"][i, :a], o["keys"][i, :a]), f"{label}: keys inst {i}"
            assert np.array_equal(g["grant"][i, :a], o["grant"][i, :a]), f"{label}: grant inst {i}"
    else:
        n = o["n_active"]
        mask = np.arange(g["order"].shape[1])[None, :] < n[:, None]
        assert np.array_equal(np.where(mask, g["order"], 0), np.where(mask, o["order"], 0)), f"{label}: order"
        assert np.array_equal(np.where(mask, g["keys"], 0), np.where(mask, o["keys"], 0)), f"{label}: keys"
        assert np.array_equal(np.where(mask, g["grant"], 0), np.where(mask, o["grant"], 0)), f"{label}: grant"
        assert np.array_equal(g["tier_off"], o["tier_off"]), f"{label}: tier offsets"


@pytest.mark.parametrize("n", [4_194_304, 16_000_000])
def test_prefix_step_size_sweep_parity(n):
    rec = tracegen.cfg4_records(n)
    cfg, ip = tracegen.PRESET_CFG4, tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    del rec
    t0 = 65536
    for k in range(4):
        o = st.step(t0 + k)
        assert o["rc"] == 0
        g = s.step_result(s.step(t0 + k, prefix=True))
        check_step(g, o, 1, f"prefix {n} step {k}", True)
        assert int(g["admitted"][0]) > 0
    assert np.array_equal(s.slots(0), st.slots(0)), f"prefix {n}: slot state"
    assert s.ledger(0) == st.ledger(0)
    s.close()
    st.close()


def batched_records(n_inst, ma, varied):
    if not varied:
        r = tracegen.cfg4_records(ma, n_running=16, n_swapped=16, n_paused=4)
        return [r] * n_inst
    sets = [tracegen.cfg4_records(ma, seed=100 + k, n_running=8 * (k + 1), n_swapped=4 * k, n_paused=k)
            for k in range(8)]
    return [sets[i % 8] for i in range(n_inst)]


@pytest.mark.parametrize("prefix", [False, True])
@pytest.mark.parametrize("varied", [False, True])
def test_batched_4096x2048_parity(prefix, varied):
    """bench.py step_multi: 4,096 instances x 2,048 slots, one call per step
    (varied=False is the bench's exact input; varied=True cycles 8 record
    sets and 4 target_max values so instances differ)."""
    n_inst, ma = 4096, 2048
    cfg = tracegen.PRESET_CFG4
    ip = tracegen.inst_params(n_inst) if not varied else \
        tracegen.inst_params(n_inst, target_max=np.array([250, 500, 750, 1000])[np.arange(n_inst) % 4],
                             alpha=np.array([0.0, 4.6e6, 4.6e7, 4.6e8])[(np.arange(n_inst) // 4) % 4])
    recs = batched_records(n_inst, ma, varied)
    st = oracle.Step(cfg, ip, ma)
    s = aug.Scheduler(cfg, ip, n_inst, ma)
    for i in range(n_inst):
        assert st.enqueue(i, recs[i]) == 0
        s.enqueue(i, recs[i])
    t0 = 65536
    for k in range(3):
        o = st.step(t0 + k)
        assert o["rc"] == 0
        g = s.step_result(s.step(t0 + k, prefix=prefix))
        check_step(g, o, n_inst, f"batched prefix={prefix} varied={varied} step {k}", prefix)
    for i in (0, 1, 2, 3, 4095):
        assert np.array_equal(s.slots(i), st.slots(i)), f"slots inst {i}"
    s.close()
    st.close()


def test_cfg5_through_iteration_37500():
    """The driver's bench windows: 25 x 1,500 iterations with resume; a
    sample of 32 instances (every parameter point of the first trace and 16
    spread over the set) equals the oracle run to iteration 37,500."""
    import argparse
    import bench
    from test_gpu_simulate import assert_equal_records
    args = argparse.Namespace(workload="cfg5", instances=65536, scaling="strong")
    tr, ip, tid, ma, _, _ = bench.workload(args, 0, 1)
    n = len(tid)
    s = aug.Scheduler(tracegen.PRESET_7B, ip, n, ma)
    dt = aug.DeviceTraces(tr)
    tid_d = torch.from_numpy(tid.astype(np.int32)).cuda()
    out = torch.empty(n * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    W = 1500
    for k in range(25):
        s.simulate(dt, tid_d, (k + 1) * W, out=out, resume=k > 0)
    g = aug.results_to_numpy(out)
    s.sync()
    s.close()
    sample = np.concatenate([np.arange(16), np.linspace(16, n - 1, 16).astype(np.int64)])
    sub = {k: v[sample] for k, v in ip.items()}
    o = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[sample], max_iters=25 * W)
    assert_equal_records(g[sample], o, "cfg5 @37,500")
    d = [oracle.as_dict(x) for x in o]
    assert max(x["final_t"] for x in d) >= 25 * W - 1 or all(x["completed"] == x["n_requests"] for x in d)


@pytest.mark.parametrize("n", [1_000_000, 4_194_304])
def test_full_step_single_queue_parity(n):
    """augsched_step (the full order, one cooperative kernel) on one queue at
    the bench's sizes: 1M (each CTA's chunk fits one sub-tile: kept in
    registers) and 4M (several sub-tiles per CTA), three steps; order, keys,
    grants, tier offsets and the slot state equal the oracle's."""
    rec = tracegen.cfg4_records(n)
    cfg, ip = tracegen.PRESET_CFG4, tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    s = aug.Scheduler(cfg, ip, 1, n)
    s.enqueue(0, rec)
    del rec
    t0 = 65536
    for k in range(3):
        o = st.step(t0 + k)
        assert o["rc"] == 0
        g = s.step_result(s.step(t0 + k))
        check_step(g, o, 1, f"full {n} step {k}", False)
    assert np.array_equal(s.slots(0), st.slots(0)), f"full {n}: slot state"
    s.close()
    st.close()
