"""Multi-rank GPU path of SURVEY §8(e) on one B200: two ranks (one process
each, both on cuda:0, gloo collectives on host copies) each run the CUDA
simulate kernel on their strided shard of one instance set, all-gather the
fixed-size result records and un-permute them; the result must equal a
single-process GPU run of the whole set byte for byte, and the oracle on a
sample.  A second test runs bench.py itself under torchrun with two ranks
(strong scaling) and checks its JSON line and its sampled 1-GPU
verification."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_INST, W, WINDOWS = 96, 400, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    tr = tracegen.gen_traces(6, 600, [2.0, 3.0, 4.0, 5.0, 3.0, 2.0], seed=77)
    ip = tracegen.cfg5_params(N_INST)
    tid = (np.arange(N_INST) // 16).astype(np.uint32)
    return tr, ip, tid


def _run(ip, tid, tr):
    import paper_2512_04013_b200 as aug
    s = aug.Scheduler(tracegen.PRESET_7B, ip, len(tid), 600)
    dt = aug.DeviceTraces(tr)
    tid_d = torch.from_numpy(tid.astype(np.int32)).cuda()
    out = None
    for k in range(WINDOWS):
        out = s.simulate(dt, tid_d, W * (k + 1), out=out, resume=k > 0)
    torch.cuda.synchronize()
    s.close()
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2512_04013_b200 import dist as adist
    import paper_2512_04013_b200 as aug
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, ip, tid = _workload()
        mine = adist.strided_instances(N_INST, rank, world)
        sub = {k: np.ascontiguousarray(v[mine]) for k, v in ip.items()}
        out = _run(sub, tid[mine], tr)
        m = adist.per_rank_count(N_INST, world)
        blk = torch.zeros(m * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        blk[: out.numel()] = out
        g = adist.all_gather_records(blk, world)
        if rank == 0:
            recs = g.cpu().numpy().view(aug.RESULT_DTYPE)
            q.put(adist.unpermute(recs, N_INST, world).tobytes())
    finally:
        dist.destroy_process_group()


def test_two_ranks_strided_cuda_equals_single_gpu_and_oracle():
    import torch.multiprocessing as mp
    import paper_2512_04013_b200 as aug
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    tr, ip, tid = _workload()
    one = aug.results_to_numpy(_run(ip, tid, tr))
    assert got == one.tobytes(), "2-rank gathered records differ from the 1-GPU run"
    sample = np.arange(0, N_INST, 7)
    sub = {k: v[sample] for k, v in ip.items()}
    o = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[sample], max_iters=W * WINDOWS)
    assert np.frombuffer(got, aug.RESULT_DTYPE)[sample].tobytes() == o.tobytes()


def test_bench_two_ranks_strong_scaling_line():
    """bench.py under torchrun, 2 ranks on this GPU (AUGSCHED_BENCH_BACKEND=gloo),
    strong scaling over 2,048 instances: one JSON line from rank 0 with
    n_gpus 2, the max-over-ranks timing and the gathered records equal to a
    1-GPU run on the sampled instances."""
    env = dict(os.environ, AUGSCHED_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--instances", "2048", "--window", "300", "--no-step", "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["verify"]["byte_equal_to_1gpu_run"] is True
    assert d["config"]["instances_per_gpu"] == 1024
