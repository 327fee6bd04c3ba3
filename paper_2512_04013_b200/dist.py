"""Multi-GPU plumbing for augsched_simulate (host logic only).

Simulated serving instances share no state, so the path shards
with no data-path collective.  Two layouts:

* weak scaling (bench.py default): rank r owns its own block of instances
  (trace ids offset by r * traces_per_rank); the gathered records are the
  rank blocks in rank order.
* strided (a fixed instance set split over ranks): instance i
  runs on rank i mod world, which balances parameter-dependent run lengths;
  the gathered rank blocks are un-permuted back to instance order.

The only collective is the final all-gather of the fixed-size per-instance
result records (north star), over NCCL on GPUs or gloo on CPU tests.
"""
from __future__ import annotations

import numpy as np


def strided_instances(n_inst: int, rank: int, world: int) -> np.ndarray:
    """Instance ids owned by `rank` under the strided layout."""
    return np.arange(rank, n_inst, world, dtype=np.int64)


def per_rank_count(n_inst: int, world: int) -> int:
    """Padded per-rank record count so all ranks contribute equal blocks."""
    return (n_inst + world - 1) // world


def unpermute(gathered: np.ndarray, n_inst: int, world: int) -> np.ndarray:
    """Rank-major gathered blocks (each padded to per_rank_count) -> instance order."""
    m = per_rank_count(n_inst, world)
    blocks = gathered.reshape(world, m, *gathered.shape[1:])
    out = np.empty((n_inst,) + gathered.shape[1:], gathered.dtype)
    for r in range(world):
        ids = strided_instances(n_inst, r, world)
        out[ids] = blocks[r, : len(ids)]
    return out


def weak_trace_ids(n_traces_per_rank: int, rank: int) -> np.ndarray:
    """Global trace ids of rank r's shard in the weak-scaling layout."""
    return np.arange(rank * n_traces_per_rank, (rank + 1) * n_traces_per_rank, dtype=np.int64)


def all_gather_records(local, world: int):
    """All-gather equal-size uint8 record blocks (torch tensors) over the
    default process group; NCCL uses all_gather_into_tensor, other backends
    the list form.  Returns the rank-major concatenation."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    if dist.get_backend() == "nccl":
        out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    host = local.contiguous().cpu()   # gloo gathers host tensors
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host)
    return torch.cat(parts)
