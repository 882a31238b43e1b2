"""Multi-process (world size 2, gloo, CPU) checks of the env-sharded path: each rank generates exactly
its slice of the global env inputs (no scatter needed), and the end-of-run reduction takes the MAX of
the times and the SUM of the counters — the only collective of a run."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200.shard import env_range, reduce_run_stats, split_range


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = S.make_scene("C2")
    ids = list(env_range(rank, world, 3))
    ei = S.env_inputs(sc, ids, n_steps=2)
    t, c, m = reduce_run_stats([10.0 * (rank + 1), 1.0], [rank + 1.0, 5.0], world, mins=[1e-5 * (2 - rank), float("inf")])
    out[rank] = (ids, ei.x0.copy(), ei.y0.copy(), ei.ykin.copy(), t.numpy().copy(), c.numpy().copy(), m.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    world, port = 2, 29511
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    sc = S.make_scene("C2")
    full = S.env_inputs(sc, range(6), n_steps=2)
    for r in range(world):
        ids, x0, y0, yk, t, c, m = out[r]
        assert ids == [3 * r, 3 * r + 1, 3 * r + 2]
        assert np.array_equal(x0, full.x0[3 * r:3 * r + 3])
        assert np.array_equal(y0, full.y0[3 * r:3 * r + 3])
        assert np.array_equal(yk, full.ykin[:, 3 * r:3 * r + 3])
        assert np.array_equal(t, [20.0, 1.0])            # MAX over ranks
        assert np.array_equal(c, [3.0, 10.0])            # SUM over ranks
        assert np.array_equal(m, [1e-5, float("inf")])   # MIN over ranks (min contact distance)


def test_split_ranges_cover_exactly():
    for total in (7, 1024, 4096):
        for world in (1, 2, 3, 8):
            ids = [i for r in range(world) for i in split_range(r, world, total)]
            assert ids == list(range(total))
