"""GPU parity of augsched_simulate (the fused per-instance kernel) against the
CPU oracle: per-instance result records must be byte-identical (goodput
counts, busy steps, decisions, token totals, histograms)."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402


def gpu_run(cfg, ip, tr, tid, max_iters=2**32, windows=None):
    n = len(tid)
    ma = int(max(tr.trace_len(i) for i in range(tr.n_traces)))
    s = aug.Scheduler(cfg, ip, n, max(ma, 1))
    dt = aug.DeviceTraces(tr)
    tid_d = torch.from_numpy(np.asarray(tid, np.int32)).cuda()
    if windows is None:
        out = s.simulate(dt, tid_d, max_iters)
    else:
        out = None
        for k, w in enumerate(windows):
            out = s.simulate(dt, tid_d, w, resume=k > 0)
    res = aug.results_to_numpy(out)
    s.sync()
    launches = s.launches
    s.close()
    return res, launches


def assert_equal_records(g, o, label=""):
    assert g.dtype.itemsize == o.dtype.itemsize
    for i in range(len(o)):
        gd, od = aug.as_dict(g[i]), oracle.as_dict(o[i])
        for k in oracle.FIELDS:
            assert gd[k] == od[k], f"{label} instance {i} field {k}: gpu {gd[k]} oracle {od[k]}"
        assert np.array_equal(gd["hist_ttft"], od["hist_ttft"]), f"{label} {i} hist_ttft"
        assert np.array_equal(gd["hist_norm"], od["hist_norm"]), f"{label} {i} hist_norm"
    assert g.tobytes() == o.tobytes()


def golden(reqs, B, cap, ranking=0):
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, l_static=B, ranking=ranking)
    tr = tracegen.from_requests([reqs])
    return cfg, ip, tr


def R(arr, l_pre, segs):
    return {"arr": arr, "l_pre": l_pre,
            "segs": [(s[0], s[0], 0, 0.0, 0) if len(s) == 1 else (s[0], s[0], s[1], s[2], s[3]) for s in segs]}


GOLDENS = {
    "G4": ([R(0, 10, [(5,)])], 15, 10**6, 0),
    "G5": ([R(0, 10, [(2, 300_000, 0.3, 5), (1,)])], 100, 1000, 0),
    "G6": ([R(0, 10, [(10,)]), R(0, 10, [(10,)])], 20, 30, 0),
    "G7": ([R(0, 10, [(1, 5_000_000, 0.0, 2), (1,)]), R(300_000, 25, [(1,)])], 30, 30, 0),
    "G8": ([R(0, 3, [(2,)]), R(0, 3, [(2,)])], 1, 10**6, 1),
}


@pytest.mark.parametrize("name", list(GOLDENS))
def test_goldens_gpu(name):
    reqs, B, cap, rk = GOLDENS[name]
    cfg, ip, tr = golden(reqs, B, cap, rk)
    g, _ = gpu_run(cfg, ip, tr, [0])
    o = oracle.simulate(cfg, ip, tr, [0])
    assert_equal_records(g, o, name)


def test_cfg1_parity():
    """Config 1: 200 requests at 4 req/s, 7B preset; AugServe+dynamic and
    FCFS+static 500."""
    tr = tracegen.gen_traces(1, 200, [4.0], seed=1)
    ip = tracegen.inst_params(2, ranking=[0, 1], budget_mode=[0, 1], l_static=500)
    g, launches = gpu_run(tracegen.PRESET_7B, ip, tr, [0, 0])
    o = oracle.simulate(tracegen.PRESET_7B, ip, tr, [0, 0])
    assert launches >= 1
    assert_equal_records(g, o, "cfg1")


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_random_mixed_parity(seed):
    """Small traces across every ranking / budget / policy mode, alpha and
    gamma values, tiny memory (frequent eviction/demotion) and no-call
    requests."""
    rng = np.random.default_rng(seed)
    tr = tracegen.gen_traces(6, 300, [1.0, 3.0, 6.0, 10.0, 20.0, 40.0], seed=seed, p_nocall=0.25)
    n = 48
    ip = tracegen.inst_params(
        n, ranking=rng.integers(0, 3, n), rank_seed=rng.integers(0, 2**32, n), budget_mode=rng.integers(0, 2, n),
        policy_mode=rng.integers(0, 4, n), target_max=rng.integers(1, 3000, n),
        l_static=rng.integers(0, 3000, n), alpha=rng.choice([0.0, 1e3, 4.6e7, 1e12], n),
        slo_ttft_ticks=rng.integers(10**5, 10**7, n))
    tid = rng.integers(0, 6, n).astype(np.uint32)
    for cfg in (tracegen.PRESET_7B, dict(tracegen.PRESET_7B, g_total=12_100_000_000 + 2**30 + 2**29 + 3_000 * 458752,
                                          gamma_num=1, gamma_den=3)):
        # B can be 0 (l_static 0, tiny target_max): bound the run
        g, _ = gpu_run(cfg, ip, tr, tid, max_iters=60_000)
        o = oracle.simulate(cfg, ip, tr, tid, max_iters=60_000)
        assert_equal_records(g, o, f"seed{seed}")


def test_resume_windows_equal_full_run():
    tr = tracegen.gen_traces(2, 400, [4.0, 6.0], seed=8)
    ip = tracegen.inst_params(4, alpha=[0.0, 4.6e7, 0.0, 4.6e7])
    tid = [0, 0, 1, 1]
    full, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid)
    win, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid, windows=[500, 1234, 5000, 2**32])
    assert full.tobytes() == win.tobytes()
    cut, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid, max_iters=3000)
    o = oracle.simulate(tracegen.PRESET_7B, ip, tr, tid, max_iters=3000)
    assert_equal_records(cut, o, "cut")


def test_host_path_equals_device_path():
    tr = tracegen.gen_traces(3, 250, [2.0, 4.0, 8.0], seed=9)
    ip = tracegen.inst_params(6)
    tid = np.array([0, 1, 2, 0, 1, 2], np.uint32)
    dev, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid)
    s = aug.Scheduler(tracegen.PRESET_7B, ip, 6, 250)
    host = s.simulate_host(tr, tid)
    s.close()
    assert dev.tobytes() == host.tobytes()


def test_capacity_error():
    tr = tracegen.gen_traces(1, 100, [4.0], seed=1)
    s = aug.Scheduler(tracegen.PRESET_7B, tracegen.inst_params(1), 1, 50)
    with pytest.raises(aug.AugschedError) as e:
        s.simulate_host(tr, [0])
    assert e.value.code == aug.E_CAPACITY
    s.close()


def test_cfg3_sampled_parity():
    """Config 3: 4,096 instances (64 target_max x 64 TTFT SLOs) on one
    2,000-request trace; GPU runs all, the oracle a sample; plus the R30
    invariant (SLO changes classification only) over all GPU records."""
    tr = tracegen.gen_traces(1, 2000, [4.0], seed=3)
    ip = tracegen.cfg3_params()
    n = 4096
    tid = np.zeros(n, np.uint32)
    g, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid)
    sample = np.arange(0, n, 257)
    sub = {k: v[sample] for k, v in ip.items()}
    o = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[sample])
    assert_equal_records(g[sample], o, "cfg3")
    f = g["f"].reshape(64, 64, -1)
    slo_fields = [oracle.FIELDS.index("slo_ok"), oracle.FIELDS.index("slo_ok_5x")]
    keep = [i for i in range(len(oracle.FIELDS)) if i not in slo_fields]
    assert (f[:, :, keep] == f[:, :1, keep]).all()          # schedules identical across SLOs
    assert (np.diff(f[:, :, slo_fields[0]].astype(np.int64), axis=1) >= 0).all()


def test_cfg2_parity():
    """Config 2: one instance per request rate 1..8 req/s, 10,000 requests
    each, full math/QA/web/chatbot tool mix (seed 2).
    Every record byte-identical to the oracle's."""
    tr = tracegen.gen_traces(8, 10_000, [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0], seed=2)
    ip = tracegen.inst_params(8)
    tid = np.arange(8, dtype=np.uint32)
    g, _ = gpu_run(tracegen.PRESET_7B, ip, tr, tid)
    o = oracle.simulate(tracegen.PRESET_7B, ip, tr, tid, threads=8)
    assert_equal_records(g, o, "cfg2")


def test_cfg5_bench_launch_sampled_parity():
    """Config 5 at full size in the launch configuration bench.py times:
    65,536 instances of 5,000-request traces, advanced in 1,500-iteration
    resumable windows; a sample of instances is re-simulated by the oracle
    for the same number of iterations and compared record by record."""
    import bench
    import argparse
    args = argparse.Namespace(workload="cfg5", instances=65536, scaling="strong")
    tr, ip, tid, ma, _, _ = bench.workload(args, 0, 1)
    n = len(tid)
    s = aug.Scheduler(tracegen.PRESET_7B, ip, n, ma)
    dt = aug.DeviceTraces(tr)
    tid_d = torch.from_numpy(tid.astype(np.int32)).cuda()
    out = torch.empty(n * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    W = 1500
    for k in range(2):
        s.simulate(dt, tid_d, (k + 1) * W, out=out, resume=k > 0)
    g = aug.results_to_numpy(out)
    s.sync()
    s.close()
    sample = np.concatenate([np.arange(16), np.arange(16, n, 4099)])
    sub = {k: v[sample] for k, v in ip.items()}
    o = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[sample], max_iters=2 * W, threads=16)
    assert_equal_records(g[sample], o, "cfg5")


def test_edge_cases_parity():
    """Degenerate inputs against the oracle: an empty trace, a static limit of
    0 (nothing is ever admitted, bounded by max_iters), a request with 255
    segments (the largest n_seg), many one-token prompts under a large limit
    (more than 32 admitted waiting entries per step: the radix-select
    fallback of the pop rounds) and tight memory with a large running set
    (more than 64 eviction candidates: the radix-select eviction)."""
    reqs_empty = []
    reqs_many_segs = [R(0, 5, [(1, 10_000, 0.01, 1)] * 254 + [(2,)])]
    reqs_tiny = [R(1000 * i, 1, [(3,)]) for i in range(400)]
    reqs_big_run = [R(0, 40, [(30,)]) for _ in range(160)]
    tr = tracegen.from_requests([reqs_empty, reqs_many_segs, reqs_tiny, reqs_big_run])
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + 3000, g_model=1000)   # cap 3,000 tokens
    ip = tracegen.inst_params(6, base=tracegen.INST_G0, budget_mode=[1, 1, 1, 0, 1, 0],
                              l_static=[50, 0, 100, 0, 2000, 0], target_max=[50, 50, 50, 50, 50, 3000],
                              alpha=[0.0, 0.0, 0.0, 2.0, 0.0, 1.0])
    tid = np.array([0, 1, 1, 2, 2, 3], np.uint32)
    g, _ = gpu_run(cfg, ip, tr, tid, max_iters=5000)
    o = oracle.simulate(cfg, ip, tr, tid, max_iters=5000)
    assert_equal_records(g, o, "edge")
    d = [oracle.as_dict(x) for x in o]
    assert d[0]["n_requests"] == 0 and d[0]["busy_steps"] == 0
    assert d[1]["completed"] == 0 and d[1]["decisions"] > 0          # limit 0
    assert d[2]["completed"] == 1                                     # 255 segments
    assert d[3]["completed"] == 400 and d[4]["completed"] == 400      # tiny prompts
    assert d[5]["evictions"] > 0


def test_n_seg_above_255_is_rejected():
    tr = tracegen.from_requests([[R(0, 5, [(1, 1000, 0.0, 1)] * 255 + [(1,)])]])
    s = aug.Scheduler(tracegen.PRESET_G0, tracegen.inst_params(1, base=tracegen.INST_G0), 1, 4)
    with pytest.raises(aug.AugschedError) as e:
        s.simulate_host(tr, [0])
    assert e.value.code == aug.E_INVALID
    s.close()


def test_max_iters_above_2_32_is_rejected():
    """Last-scheduled iterations are stored as u32 (R14): max_iters > 2^32
    is rejected instead of silently wrapping."""
    tr = tracegen.from_requests([[R(0, 5, [(2,)])]])
    s = aug.Scheduler(tracegen.PRESET_G0, tracegen.inst_params(1, base=tracegen.INST_G0), 1, 4)
    with pytest.raises(aug.AugschedError) as e:
        s.simulate_host(tr, [0], max_iters=2**32 + 1)
    assert e.value.code == aug.E_INVALID
    s.simulate_host(tr, [0], max_iters=2**32)
    s.close()
