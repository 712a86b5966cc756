"""CPU (gloo, world size 2) check of bench.py's multi-rank plumbing for the
batched configs: every rank draws the SAME seeded batch and prices the share
amtc_batch_shard_plan deals it (strong scaling); the step time is the MAX over
ranks."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    w, r, local, pg = bench.setup_dist()
    assert (w, r) == (world, rank)
    from paper_1110_2477_b200 import api
    b, N, _ = bench.workload(4)
    rank_of, _ = api.batch_shard_plan(b, N, w)
    mine = int((rank_of == r).sum())
    t = bench.max_over_ranks(float(r + 1), pg, "cpu")
    s = bench.sum_over_ranks(float(mine), pg, "cpu")
    q.put((r, t, s, float(b.K[0]), N))
    pg.barrier()
    pg.destroy_process_group()


def test_bench_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(t == 2.0 for _, t, _, _, _ in res)          # max over ranks
    assert all(s == 16384 for _, _, s, _, _ in res)        # the shares partition ONE batch
    assert res[0][3] == res[1][3]                           # the same seeded batch on every rank
    assert all(N == 1500 for *_, N in res)
