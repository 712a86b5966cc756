"""The batched multi-GPU split (BASELINE.json north_star: "splits
options across the 8 B200s with no inter-GPU traffic except a final gather").

CPU tests of the REAL deal and gather code: the library's host-only
amtc_batch_shard_plan and paper_1110_2477_b200.dist over a gloo process group
(world size 2 and 3).  On a CPU box the per-rank pricing step is the oracle
(tests may call it); on GPUs it is the CUDA batch API -- the plan and the
gather around it are the same code."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1110_2477_b200 import api, workloads as W


def test_plan_equal_counts_and_balanced_cost():
    b = W.config4()
    for n in (1, 2, 4, 8):
        rank_of, cost = api.batch_shard_plan(b, W.CONFIG4_N, n)
        counts = np.bincount(rank_of, minlength=n)
        assert counts.sum() == len(b) and counts.max() - counts.min() <= 1   # "split evenly"
        assert cost.max() / cost.mean() < 1.01                                # snake deal balances the estimate
        assert rank_of.min() >= 0 and rank_of.max() < n


def test_plan_deterministic_and_deals_heavy_items_round_robin():
    b = W.config4(n=64)
    r1, _ = api.batch_shard_plan(b, 1500, 4)
    r2, _ = api.batch_shard_plan(b, 1500, 4)
    assert (r1 == r2).all()
    # the four most expensive options (calls / bulls at the largest k/h) land on four different ranks
    h = b.sigma * np.sqrt(b.T / 1500)
    est = 2 + 4.0 * (b.kind != W.PUT) * b.k / h
    top = np.argsort(-est, kind="stable")[:4]
    assert sorted(r1[top]) == [0, 1, 2, 3]


def test_plan_rejects_bad_arguments():
    b = W.config4(n=8)
    with pytest.raises(ValueError):
        api.batch_shard_plan(b, 0, 2)
    with pytest.raises(ValueError):
        api.batch_shard_plan(b, 100, 0)


def _oracle_pricer(sub, N):
    import oracle as O
    out = np.zeros(len(sub), dtype=api.QUOTE_DTYPE)
    for i in range(len(sub)):
        r = sub.row(i)
        q = O.price_tc(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], r["k"], r["kind"], r["K2"]), N)
        out[i] = (q.ask, q.bid, q.status, max(q.max_kinks_ask, q.max_kinks_bid))
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_1110_2477_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = W.random_small(23, seed=77, k_max=0.03)   # odd size: ragged per-rank counts
    quotes, idx = D.price_batch_sharded(b, 24, rank, world, pricer=_oracle_pricer)
    q.put((rank, quotes.tobytes(), idx.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + world * 7 + os.getpid() % 500
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    b = W.random_small(23, seed=77, k_max=0.03)
    ref = _oracle_pricer(b, 24)
    for rank, qb, idx in res:
        got = np.frombuffer(qb, dtype=api.QUOTE_DTYPE)
        assert (got["ask"] == ref["ask"]).all() and (got["bid"] == ref["bid"]).all()   # batch order restored
    # the ranks' index sets partition the batch
    allidx = sorted(i for _, _, idx in res for i in idx)
    assert allidx == list(range(len(b)))
