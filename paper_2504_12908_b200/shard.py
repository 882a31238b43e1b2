"""Env sharding across GPUs: contiguous global env-id ranges per rank, no exchange on
the hot path, and the single end-of-run statistics reduction (max of times, sum of counters)."""
from __future__ import annotations

import torch


def env_range(rank: int, world: int, envs_per_rank: int):
    """Weak scaling: rank r owns global env ids [r·E, (r+1)·E)."""
    return range(rank * envs_per_rank, (rank + 1) * envs_per_rank)


def split_range(rank: int, world: int, total: int):
    """Strong scaling split: [⌊rE/G⌋, ⌊(r+1)E/G⌋)."""
    return range(rank * total // world, (rank + 1) * total // world)


def reduce_run_stats(times_ms, counters, world: int, device=None, mins=None):
    """All-reduce the timed-region stats: MAX over ranks of the times, SUM of the counters and MIN of
    `mins` (e.g. the minimum contact distance, the intersection-free certificate).  Works on any
    backend (nccl on the GPU box with a CUDA `device`, gloo in the CPU tests).  Returns (times,
    counters) or, when `mins` is given, (times, counters, mins)."""
    t = torch.as_tensor(times_ms, dtype=torch.float64, device=device)
    c = torch.as_tensor(counters, dtype=torch.float64, device=device)
    m = torch.as_tensor(mins if mins is not None else [0.0], dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        if mins is not None:
            dist.all_reduce(m, op=dist.ReduceOp.MIN)
    if mins is None:
        return t.cpu(), c.cpu()
    return t.cpu(), c.cpu(), m.cpu()
