"""Multi-process (world size 2, gloo on CPU) tests of the sharding and the
final record gather: the records of a strided shard set, gathered and
un-permuted, equal the single-process records byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tracegen
from paper_2512_04013_b200 import dist as adist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_inst, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = tracegen.gen_traces(3, 60, [3.0, 6.0, 9.0], seed=21)
        ip = tracegen.inst_params(n_inst, target_max=np.arange(n_inst) * 37 + 100,
                                  alpha=np.where(np.arange(n_inst) % 2, 4.6e7, 0.0))
        tid = (np.arange(n_inst) % 3).astype(np.uint32)
        mine = adist.strided_instances(n_inst, rank, world)
        m = adist.per_rank_count(n_inst, world)
        sub = {k: v[mine] for k, v in ip.items()}
        # the per-rank compute (here the CPU oracle stands in for the GPU kernel)
        res = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[mine], threads=1)
        blk = np.zeros(m, oracle.RESULT_DTYPE)
        blk[: len(mine)] = res
        t = torch.from_numpy(blk.view(np.uint8).copy())
        g = adist.all_gather_records(t, world)
        if rank == 0:
            gathered = g.numpy().view(oracle.RESULT_DTYPE)
            q.put(adist.unpermute(gathered, n_inst, world).tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_inst", [7, 8])
def test_strided_shard_gather_unpermute_equals_single_process(n_inst):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_inst, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tr = tracegen.gen_traces(3, 60, [3.0, 6.0, 9.0], seed=21)
    ip = tracegen.inst_params(n_inst, target_max=np.arange(n_inst) * 37 + 100,
                              alpha=np.where(np.arange(n_inst) % 2, 4.6e7, 0.0))
    tid = (np.arange(n_inst) % 3).astype(np.uint32)
    ref = oracle.simulate(tracegen.PRESET_7B, ip, tr, tid, threads=1)
    assert got == ref.tobytes()


def test_unpermute_and_weak_ids():
    n, w = 10, 4
    owner = np.concatenate([adist.strided_instances(n, r, w) for r in range(w)])
    assert sorted(owner.tolist()) == list(range(n))
    m = adist.per_rank_count(n, w)
    blocks = np.full((w, m), -1)
    for r in range(w):
        ids = adist.strided_instances(n, r, w)
        blocks[r, : len(ids)] = ids * 10
    assert adist.unpermute(blocks.reshape(-1), n, w).tolist() == [i * 10 for i in range(n)]
    assert adist.weak_trace_ids(4, 2).tolist() == [8, 9, 10, 11]
