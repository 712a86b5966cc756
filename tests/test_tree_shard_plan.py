"""CPU check of the strip partition of the sharded transaction-cost tree
(amtc_tree_shard_plan, host-only part of libamtc): contiguous ranges that cover
every strip once, rank 0 holds the root strip, and the per-rank work (strip s
carries N - 32 s + 1 levels) is balanced to within one strip."""
import pytest


@pytest.mark.parametrize("N,n", [(64, 2), (1000, 2), (8000, 2), (8000, 4), (8000, 8), (2000, 8), (300, 8)])
def test_shard_plan(N, n):
    from paper_1110_2477_b200 import api
    lo = api.tree_shard_plan(N, n)
    S = N // 32 + 1
    assert lo[0] == 0 and lo[-1] == S
    assert all(a <= b for a, b in zip(lo, lo[1:]))
    work = lambda s: N - 32 * s + 1
    per = [sum(work(s) for s in range(lo[g], lo[g + 1])) for g in range(n)]
    total = sum(work(s) for s in range(S))
    assert sum(per) == total
    assert max(per) - total / n <= work(0) + 1
