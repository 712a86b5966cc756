"""GPU parity of the single large-tree path (config 5a) and of the sharded
entry point on one rank, through the C-ABI, against the CPU oracle."""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_1110_2477_b200 import workloads as W

pytestmark = pytest.mark.gpu
from tolerance import close  # noqa: E402  (1e-9 relative or the A19 rounding floor 4 N eps S0)


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available()
    from paper_1110_2477_b200 import api as A
    A.lib()
    return A


def _close(g, o, N):
    return close(g, o, N)


CASES = [(O.PUT, 100.0, 0.0), (O.CALL, 95.0, 0.0), (O.BULL, 90.0, 110.0)]


# band edges: 128 levels per band, 384 output columns per warp
@pytest.mark.parametrize("N", [1, 2, 127, 128, 129, 383, 384, 385, 511, 1000, 5001])
@pytest.mark.parametrize("case", range(3))
def test_crr_tree_matches_oracle(api, N, case):
    kind, K, K2 = CASES[case]
    g = api.price_crr_tree(100.0, K, 0.8, 0.3, 0.04, N, kind, K2)
    o = O.price_crr(O.Option(100.0, K, 0.8, 0.3, 0.04, 0.0, kind, K2), N)
    assert _close(g, o, N), (N, kind, g, o)


# every sweep shape of the single-tree path (testing hook): 1 one launch per
# band, 2..5 the wavefront kernel with (M, D) = (16, 256), (8, 128), (12, 128),
# (8, 64): N around the band height D and the slot width 32 M - D
@pytest.mark.parametrize("shape", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("N", [1, 63, 64, 65, 128, 129, 255, 256, 257, 1000, 4097, 20011])
def test_crr_tree_shapes_match_oracle(api, shape, N):
    try:
        api.debug_set_tree_shape(shape)
        for case in range(3):
            kind, K, K2 = CASES[case]
            g = api.price_crr_tree(100.0, K, 0.8, 0.3, 0.04, N, kind, K2)
            o = O.price_crr(O.Option(100.0, K, 0.8, 0.3, 0.04, 0.0, kind, K2), N)
            assert _close(g, o, N), (shape, N, kind, g, o)
        g = api.price_crr_tree(100.0, 100.0, 0.8, 0.3, 0.04, N, O.PUT, flags=api.EUROPEAN)
        o = O.price_crr(O.Option(100.0, 100.0, 0.8, 0.3, 0.04, 0.0, O.PUT, american=False), N)
        assert _close(g, o, N), (shape, N, "european", g, o)
    finally:
        api.debug_set_tree_shape(0)


def test_crr_tree_wave_repeatable(api):
    """The wavefront's progress counters are reset per call: repeated calls at
    different N (slot counts shrinking and growing) give bitwise equal prices."""
    vals = {}
    for rep in range(3):
        for N in (30000, 777, 100000, 5):
            g = api.price_crr_tree(100.0, 100.0, 1.0, 0.3, 0.05, N, O.PUT)
            if rep == 0:
                vals[N] = g
            assert g == vals[N], (rep, N, g, vals[N])


def test_crr_tree_equals_batch_kernel(api):
    b = W.random_small(16, seed=77, k_max=0.0)
    N = 700
    batch = api.price_crr_batch_host(b, N)
    for i in range(len(b)):
        r = b.row(i)
        g = api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, r["kind"], r["K2"])
        assert _close(g, batch[i], N), (i, g, batch[i])


def test_appendix_put_13906(api):
    """American put K=S0=100, T=3, sigma=0.3, R=0.06 -> 13.906 (reading A16: N=40000)."""
    a = W.appendix_put().row(0)
    g = api.price_crr_tree(a["S0"], a["K"], a["T"], a["sigma"], a["R"], 40000, O.PUT)
    assert abs(g - 13.906) <= 5e-4
    o = O.price_crr(O.Option(a["S0"], a["K"], a["T"], a["sigma"], a["R"], 0.0, O.PUT), 40000)
    assert _close(g, o, 40000), (g, o)


def test_config5a_full_size(api):
    """BASELINE config 5a: put S0=K=100, T=1, sigma=0.3, R=0.05, k=0, N=100000."""
    r = W.config5a().row(0)
    g = api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], W.CONFIG5A_N, O.PUT)
    o = O.price_crr(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], 0.0, O.PUT), W.CONFIG5A_N)
    assert _close(g, o, W.CONFIG5A_N), (g, o)


def test_tree_invalid_inputs(api):
    with pytest.raises(ValueError):
        api.price_crr_tree(-1.0, 100.0, 1.0, 0.2, 0.05, 100)
    with pytest.raises(ValueError):  # d < r < u violated
        api.price_crr_tree(100.0, 100.0, 1.0, 0.01, 5.0, 10)


def test_sharded_one_rank_nccl(api):
    """amtc_price_tree_sharded over a one-rank NCCL communicator: the same
    numbers as the single-GPU tree (k = 0) and the single-option TC call (k > 0)."""
    comm = api.comm_init(api.comm_unique_id(), 1, 0)
    try:
        for N in (130, 2000):
            q = api.price_tree_sharded(100.0, 100.0, 1.0, 0.3, 0.05, N, 0.0, O.PUT, comm=comm, rank=0, nranks=1)
            o = O.price_crr(O.Option(100.0, 100.0, 1.0, 0.3, 0.05, 0.0, O.PUT), N)
            assert q["status"] == 0 and _close(q["ask"], o, N) and q["bid"] == q["ask"], (q, o)
        # k > 0 through the sharded transaction-cost path (one rank: no peer)
        for N, kind, K, k in ((200, O.PUT, 100.0, 0.005), (300, O.CALL, 95.0, 0.02), (1000, O.PUT, 100.0, 0.005)):
            q = api.price_tree_sharded(100.0, K, 1.0, 0.3, 0.05, N, k, kind, comm=comm, rank=0, nranks=1)
            o = O.price_tc(O.Option(100.0, K, 1.0, 0.3, 0.05, k, kind), N)
            assert q["status"] == 0 and _close(q["ask"], o.ask, N) and _close(q["bid"], o.bid, N), (N, q, o)
    finally:
        api.comm_destroy(comm)
    # no communicator, one rank
    q = api.price_tree_sharded(100.0, 100.0, 1.0, 0.3, 0.05, 300, 0.0, O.PUT)
    assert q["status"] == 0
    # several ranks need a communicator
    q = api.price_tree_sharded(100.0, 100.0, 1.0, 0.3, 0.05, 300, 0.005, O.PUT, comm=None, rank=0, nranks=2)
    assert q["status"] == 1 and math.isnan(q["ask"])


def test_very_long_tree_1e6(api):
    """a very-long-dated k=0 tree, N = 10^6 (8 MB level,
    7813 bands), converges to the paper's 13.906 (reading A16) and agrees
    with N = 40000 to the paper's 3 decimals."""
    a = W.appendix_put().row(0)
    g6 = api.price_crr_tree(a["S0"], a["K"], a["T"], a["sigma"], a["R"], 1_000_000, O.PUT)
    g4 = api.price_crr_tree(a["S0"], a["K"], a["T"], a["sigma"], a["R"], 40_000, O.PUT)
    assert abs(g6 - 13.906) <= 5e-4 and abs(g6 - g4) <= 5e-4, (g6, g4)


def _tree_goldens():
    """N of every cached oracle value present under tests/golden/ (written only by
    scripts/make_tree_refs.py; N = 2e5 is committed, 4e5 takes ~48 CPU-minutes)."""
    import glob
    import re
    pat = os.path.join(os.path.dirname(__file__), "golden", "oracle_tree_appendix_put_N*.json")
    return sorted(int(re.search(r"_N(\d+)\.json$", f).group(1)) for f in glob.glob(pat))


@pytest.mark.parametrize("N", _tree_goldens())
def test_long_tree_against_oracle_golden(api, N):
    """SURVEY 8(f) NEXT #4 backed by the oracle beyond the suite's own reach: the
    appendix put at N = 2e5 and 4e5 against oracle values cached by
    scripts/make_tree_refs.py (plain scalar CRR, ~12 / 48 CPU-minutes each)."""
    import json
    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_tree_appendix_put_N{N}.json")
    ref = json.load(open(path))
    a = W.appendix_put().row(0)
    assert (ref["S0"], ref["K"], ref["T"], ref["sigma"], ref["R"]) == (a["S0"], a["K"], a["T"], a["sigma"], a["R"])
    g = api.price_crr_tree(a["S0"], a["K"], a["T"], a["sigma"], a["R"], N, O.PUT)
    assert _close(g, ref["price"], N), (g, ref["price"])
