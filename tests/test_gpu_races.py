"""Race / synchronisation checks of the transaction-cost solvers without
compute-sanitizer (closed on this GPU pool: profiles/r02_sanitizer_attempt.log).

Every node function is computed by a fixed algorithm from fixed inputs,
whichever warp runs it: a tier-3 node claimed by any warp of the CTA (mailbox,
claim bits, `done` counter), a strip handed over through a carry column (in
shared memory, or through HBM progress counters in split mode), the light and
full kernels running side by side on two streams.  So the quotes are a pure
function of the batch, and any race in those protocols (a read of a mailbox
or carry before it is published, a slot reused while still read) shows up as
a run-to-run difference.  These tests run each schedule-sensitive mode several
times under maximal contention (tier 3 forced onto small nodes so that warps
claim each other's nodes on almost every level) and require BITWISE equal
quotes across runs, plus parity with the oracle on a sample."""
import numpy as np
import pytest

import oracle as O
from paper_1110_2477_b200 import workloads as W
from tolerance import check_arrays

pytestmark = pytest.mark.gpu

N = 300


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available()
    from paper_1110_2477_b200 import api as A
    A.lib()
    yield A
    A.debug_set_heavy_threshold(-1)
    A.debug_set_split_mode(-1)
    A.debug_set_light_kernel(1)
    A.debug_set_full_kernel(0)


@pytest.fixture(scope="module")
def batch():
    """Config-4-shaped options (calls and bull spreads grow the buyer's
    sawtooth, puts stay light), 600 of them: more items than one CTA wave."""
    b = W.config4()
    idx = np.concatenate([np.nonzero(b.kind == 1)[0][:300], np.nonzero(b.kind == 2)[0][:150],
                          np.nonzero(b.kind == 0)[0][:150]])
    return b.subset(idx)


def _runs(api, cols, reps=3):
    import torch
    out = []
    for _ in range(reps):
        q, rc = api.price_american_tc_batch(cols, N)
        torch.cuda.synchronize()
        assert rc == 0
        out.append(api.quotes_to_numpy(q).copy())
    return out


def _bitwise_equal(runs):
    a = runs[0]
    for r in runs[1:]:
        for f in ("ask", "bid", "status", "max_bp"):
            assert np.array_equal(a[f].view(np.uint64) if a[f].dtype == np.float64 else a[f],
                                  r[f].view(np.uint64) if r[f].dtype == np.float64 else r[f]), f


def _oracle_sample(api, batch, q, n=40):
    idx = np.linspace(0, len(batch) - 1, n).astype(int)
    opts = [O.Option(*(batch.row(int(i))[k] for k in ("S0", "K", "T", "sigma", "R", "k", "kind", "K2")))
            for i in idx]
    want = O.price_tc_many(opts, N)
    oka, _ = check_arrays(q["ask"][idx], [w.ask for w in want], N)
    okb, _ = check_arrays(q["bid"][idx], [w.bid for w in want], N)
    assert oka.all() and okb.all()


@pytest.mark.parametrize("full", [0, 1])
@pytest.mark.parametrize("tl", [-1, 6])
def test_whole_tree_work_sharing_deterministic(api, batch, full, tl):
    """Whole-tree mode, light kernel beside the full kernel on a second stream;
    tl = 6 forces tier 3 (CTA work sharing) onto nodes with more than 6 child
    vertices, so mailboxes and claims are exercised on most levels."""
    api.debug_set_split_mode(0)
    api.debug_set_light_kernel(1)
    api.debug_set_full_kernel(full)
    api.debug_set_heavy_threshold(tl)
    runs = _runs(api, api.device_batch(batch))
    _bitwise_equal(runs)
    _oracle_sample(api, batch, runs[0])


@pytest.mark.parametrize("tl", [-1, 6])
def test_split_mode_progress_handoff_deterministic(api, batch, tl):
    """Strip-split mode: strips of one tree on different warps, pipelined
    through HBM progress counters and per-strip carry columns."""
    api.debug_set_split_mode(1)
    api.debug_set_heavy_threshold(tl)
    sub = batch.subset(np.arange(0, len(batch), 25))  # few trees: split mode applies
    runs = _runs(api, api.device_batch(sub), reps=4)
    _bitwise_equal(runs)
    _oracle_sample(api, sub, runs[0], n=len(sub))


def test_light_split_handoff_deterministic(api, batch):
    """The light kernel's split mode (light trees only: puts): cp.async-staged
    carry records behind HBM progress counters, bitwise equal over runs."""
    api.debug_set_split_mode(1)
    api.debug_set_heavy_threshold(-1)
    sub = batch.subset(np.nonzero(batch.kind == W.PUT)[0][::15])
    runs = _runs(api, api.device_batch(sub), reps=4)
    _bitwise_equal(runs)
    _oracle_sample(api, sub, runs[0], n=len(sub))


def test_modes_agree_within_tolerance(api, batch):
    """The same batch through whole-tree mode (both full kernels) and split
    mode: equal within the parity tolerance (different tiers may round
    differently, reading A20)."""
    import torch
    api.debug_set_heavy_threshold(-1)
    cols = api.device_batch(batch)
    res = []
    for split, full in ((0, 0), (0, 1), (1, 0)):
        api.debug_set_split_mode(split)
        api.debug_set_full_kernel(full)
        q, rc = api.price_american_tc_batch(cols, N)
        torch.cuda.synchronize()
        assert rc == 0
        res.append(api.quotes_to_numpy(q).copy())
    for r in res[1:]:
        assert check_arrays(r["ask"], res[0]["ask"], N)[0].all()
        assert check_arrays(r["bid"], res[0]["bid"], N)[0].all()
