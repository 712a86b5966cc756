"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Tolerance (north star): 1e-9 relative in fp64; only where
the oracle's price is below 1e-6 an absolute floor of 4 N eps S0 (reading A19
in DESIGN.md, tests/tolerance.py).  Every option in these tests has S0 = 100."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_1110_2477_b200 import workloads as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
from tolerance import check_arrays, close, floor  # noqa: E402  (1e-9 relative; A19 floor only for |o| < 1e-6)


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available()
    from paper_1110_2477_b200 import api as A
    A.lib()
    return A


def _opt(row):
    return O.Option(row["S0"], row["K"], row["T"], row["sigma"], row["R"], row["k"], row["kind"], row["K2"])


def assert_quotes(got, batch, N, want=None):
    want = want if want is not None else [O.price_tc(_opt(batch.row(i)), N) for i in range(len(batch))]
    bad = []
    for i, q in enumerate(want):
        g = got[i]
        assert g["status"] == q.status, (i, batch.row(i), g, q)
        if q.status:
            assert math.isnan(g["ask"]) and math.isnan(g["bid"])
            continue
        if not (close(g["ask"], q.ask, N) and close(g["bid"], q.bid, N)):
            bad.append((i, batch.row(i), float(g["ask"]), q.ask, float(g["bid"]), q.bid))
    assert not bad, bad[:5]


@pytest.mark.parametrize("N", [1, 2, 3, 7, 33, 130])
def test_tc_random_small(api, N):
    b = W.random_small(48, seed=1000 + N, k_max=0.05)
    got, rc = api.price_american_tc_batch_host(b, N)
    assert rc == 0
    assert_quotes(got, b, N)


def test_tc_device_batch_matches_host(api):
    import torch
    b = W.random_small(40, seed=77)
    cols = api.device_batch(b)
    out, rc = api.price_american_tc_batch(cols, 60)
    torch.cuda.synchronize()
    dev = api.quotes_to_numpy(out)
    host, rc2 = api.price_american_tc_batch_host(b, 60)
    assert rc == rc2 == 0
    np.testing.assert_array_equal(dev["ask"], host["ask"])
    np.testing.assert_array_equal(dev["bid"], host["bid"])


def test_config1_single_put(api):
    """BASELINE config 1 through the north-star single-option call."""
    for k in (0.005, 0.0):
        q = api.price_american_tc(100.0, 100.0, 0.25, 0.2, 0.1, W.CONFIG1_N, k, api.PUT)
        o = O.price_tc(O.Option(100.0, 100.0, 0.25, 0.2, 0.1, k, O.PUT), W.CONFIG1_N)
        assert q["status"] == 0
        assert close(q["ask"], o.ask, W.CONFIG1_N) and close(q["bid"], o.bid, W.CONFIG1_N), (q, o)
    crr = O.price_crr(O.Option(100.0, 100.0, 0.25, 0.2, 0.1, 0.0, O.PUT), W.CONFIG1_N)
    assert abs(q["ask"] - crr) <= 1e-9 * crr and abs(q["bid"] - crr) <= 1e-9 * crr


def test_edge_cases(api):
    # empty batch
    empty = W.random_small(0, seed=1)
    got, rc = api.price_american_tc_batch_host(empty, 10)
    assert rc == 0 and len(got) == 0
    # invalid / arbitrage options mixed with valid ones
    b = W.random_small(6, seed=5)
    b.S0[1] = -1.0
    b.k[2] = 1.0
    b.kind[3] = 9
    b.sigma[4] = 1e-4  # h tiny -> r >= u at R > 0 ?
    b.R[4] = 0.08
    got, rc = api.price_american_tc_batch_host(b, 8)
    assert got["status"][1] == 1 and got["status"][2] == 1 and got["status"][3] == 1
    assert got["status"][4] == 2
    assert rc == 2 or rc == 1
    assert_quotes(got, b, 8)
    # k = 0: lines only; equals CRR
    b0 = W.random_small(16, seed=9, k_max=0.0)
    got, rc = api.price_american_tc_batch_host(b0, 100)
    for i in range(len(b0)):
        crr = O.price_crr(_opt(b0.row(i)), 100)
        assert close(got["ask"][i], crr, 100) and close(got["bid"][i], crr, 100)


def test_config3_sweep(api):
    """BASELINE config 3: put and call, k x N sweep, single trees."""
    ref = json.load(open(os.path.join(GOLD, "oracle_config3.json")))["points"]
    bad = []
    for p in ref:
        kind = p["kind"]
        q = api.price_american_tc(100.0, 100.0, 1.0, 0.2, 0.05, p["N"], p["k"], kind)
        assert q["status"] == 0, (p, q)
        if not (close(q["ask"], p["ask"], p["N"]) and close(q["bid"], p["bid"], p["N"])):
            bad.append((p, q))
    assert not bad, bad[:3]


def _full_ref(name, batch):
    """Cached full-batch oracle values (scripts/make_full_refs.py, oracle/ only),
    keyed by the SHA-256 of the batch's SoA bytes."""
    path = os.path.join(GOLD, f"oracle_{name}_full.npz")
    assert os.path.exists(path), f"{path} missing: run scripts/make_full_refs.py {name}"
    z = np.load(path)
    assert str(z["sha256"]) == W.soa_sha256(batch), "cached oracle file does not match the workload"
    return z


def test_config4_every_option(api):
    """BASELINE config 4 at full size (16384 options, N=1500) in the bench's
    launch configuration: EVERY option's ask and bid against the cached oracle
    (the paper validates its parallel output as "exactly the same figures" as the
    sequential one)."""
    import torch
    b = W.config4()
    ref = _full_ref("config4", b)
    assert bool(ref["done"].all())
    cols = api.device_batch(b)
    out, rc = api.price_american_tc_batch(cols, W.CONFIG4_N)
    torch.cuda.synchronize()
    q = api.quotes_to_numpy(out)
    assert rc == 0, api.STATUS[rc]
    assert np.all(q["status"] == 0) and np.all(ref["status"] == 0)
    oka, fa = check_arrays(q["ask"], ref["ask"], W.CONFIG4_N, b.S0)
    okb, fb = check_arrays(q["bid"], ref["bid"], W.CONFIG4_N, b.S0)
    bad = np.nonzero(~(oka & okb))[0]
    assert bad.size == 0, [(int(i), float(q["ask"][i]), float(ref["ask"][i]), float(q["bid"][i]),
                            float(ref["bid"][i])) for i in bad[:5]]
    # the capacity audit (max_bp: the largest node function the GPU held) against
    # the oracle's largest kink count.  Representations are not unique (reading
    # A20): the GPU's value ties (A10) drop nearly collinear kinks that the
    # oracle keeps (calls at small k/h: 1 vertex vs 5-6 kinks) and keep a few
    # rounding-made ones its chord test removes (heavy buyers: up to ~20% more),
    # so only the heavy functions -- the ones the capacities exist for -- are
    # compared, within a factor that would catch a truncated or runaway function
    mk = np.maximum(ref["max_kinks_ask"], ref["max_kinks_bid"])
    assert np.all(q["max_bp"] >= 1)
    heavy = mk >= 64
    ratio = q["max_bp"][heavy] / mk[heavy]
    assert np.all((ratio >= 0.5) & (ratio <= 2.0)), (float(ratio.min()), float(ratio.max()))
    print(f"config4: 16384 x 2 prices, floor used {fa + fb} times; heavy max_bp / oracle kinks "
          f"in [{ratio.min():.3f}, {ratio.max():.3f}] over {int(heavy.sum())} options")


def test_config2_every_option(api):
    """BASELINE config 2 (65536 options, N=1024, k=0): EVERY CRR price against
    the cached oracle."""
    import torch
    b = W.config2()
    ref = _full_ref("config2", b)
    cols = api.device_batch(b)
    out = api.price_crr_batch(cols, W.CONFIG2_N)
    torch.cuda.synchronize()
    v = out.cpu().numpy()
    ok, used = check_arrays(v, ref["price"], W.CONFIG2_N, b.S0)
    bad = np.nonzero(~ok)[0]
    assert bad.size == 0, [(int(i), float(v[i]), float(ref["price"][i])) for i in bad[:5]]
    print(f"config2: 65536 prices, floor used {used} times")


@pytest.mark.parametrize("N", [1, 2, 127, 128, 129, 500, 1023, 1024, 1025, 1151, 1152])
def test_crr_small_and_ragged(api, N):
    """Register-resident CRR kernel: ragged N around the 128-node slot edges
    (N = 1024 and 1152 end the slots one node before the leaf j = N)."""
    b = W.random_small(37, seed=N)
    got = api.price_crr_batch_host(b, N)
    for i in range(len(b)):
        o = O.price_crr(_opt(b.row(i)), N)
        assert close(got[i], o, N), (i, N, got[i], o)


@pytest.mark.parametrize("N,n", [(1153, 37), (1536, 37), (2047, 20), (5000, 9), (20000, 3)])
def test_crr_batch_large_n_strip_kernel(api, N, n):
    """N above the register-resident level: the strip kernel (512-column strips,
    carry buffer per warp); Table III's frictionless trees reach N = 40,000
    (P:491-538).  Ragged strip counts, puts, calls and bull spreads
    against the oracle."""
    b = W.random_small(n, seed=N)
    got = api.price_crr_batch_host(b, N)
    for i in range(len(b)):
        o = O.price_crr(_opt(b.row(i)), N)
        assert close(got[i], o, N), (i, N, got[i], o)


def test_crr_equals_tc_at_k0(api):
    b = W.random_small(24, seed=3, k_max=0.0)
    N = 300
    crr = api.price_crr_batch_host(b, N)
    tc, rc = api.price_american_tc_batch_host(b, N)
    assert rc == 0
    assert check_arrays(tc["ask"], crr, N)[0].all() and check_arrays(tc["bid"], crr, N)[0].all()


@pytest.mark.parametrize("tl", [2, 5, 12])
def test_warp_path_forced(api, tl):
    """Force the warp-cooperative (heavy) node update onto ordinary nodes and
    check it against the oracle (the testing hook of include/amtc.h)."""
    b = W.random_small(40, seed=4000 + tl, k_max=0.08)
    ref, rc0 = api.price_american_tc_batch_host(b, 45)
    try:
        api.debug_set_heavy_threshold(tl)
        got, rc = api.price_american_tc_batch_host(b, 45)
    finally:
        api.debug_set_heavy_threshold(0)
    assert rc == 0 and rc0 == 0
    assert_quotes(got, b, 45)
    # the warp path keeps representations as lean as the lane path
    assert np.all(got["max_bp"] <= ref["max_bp"] + 4), (got["max_bp"], ref["max_bp"])


def test_heavy_sawtooth_calls(api):
    """Calls at large k/h: the buyer's node functions grow to hundreds of
    vertices (the warp path without forcing)."""
    b = W.random_small(12, seed=99, k_max=0.0)
    b.kind[:] = 1
    b.K[:] = np.linspace(90.0, 115.0, 12)
    b.k[:] = np.linspace(0.006, 0.02, 12)
    b.T[:] = 0.6
    b.sigma[:] = 0.3
    N = 400
    got, rc = api.price_american_tc_batch_host(b, N)
    assert rc == 0
    assert got["max_bp"].max() > 64  # the warp path ran
    want = [O.price_tc(_opt(b.row(i)), N) for i in range(len(b))]
    assert_quotes(got, b, N, want)
    # no representation bloat: vertex counts as in the oracle (kinks + 1), small slack
    for i, q in enumerate(want):
        assert got["max_bp"][i] <= 1.1 * (max(q.max_kinks_ask, q.max_kinks_bid) + 1) + 4, (i, got["max_bp"][i], q)


@pytest.mark.parametrize("N", [64, 97, 300])
def test_split_mode_matches_oracle(api, N):
    """Strip-split mode (the strips of one tree on different warps, pipelined
    through progress counters) against the oracle and against whole-tree mode."""
    b = W.random_small(6, seed=5000 + N, k_max=0.05)
    try:
        api.debug_set_split_mode(1)
        got, rc = api.price_american_tc_batch_host(b, N)
        api.debug_set_split_mode(0)
        ref, rc0 = api.price_american_tc_batch_host(b, N)
    finally:
        api.debug_set_split_mode(-1)
    assert rc == 0 and rc0 == 0
    assert_quotes(got, b, N)
    np.testing.assert_allclose(got["ask"], ref["ask"], rtol=1e-12, atol=floor(N))
    np.testing.assert_allclose(got["bid"], ref["bid"], rtol=1e-12, atol=floor(N))


@pytest.mark.parametrize("N", [64, 95, 97, 300])
@pytest.mark.parametrize("light_split", [1, 0])
def test_split_mode_light_trees(api, N, light_split):
    """A batch of light trees only (puts: both parties' functions stay within the
    light kernel's 6-vertex slots) in split mode: by default on the light
    kernel's split variant (carry records staged one level ahead through
    per-(tree, strip) columns and progress counters), else on the strip
    kernel's split mode; both against the oracle, ragged last strips
    included (N = 95, 97)."""
    b = W.random_small(40, seed=5100 + N, k_max=0.05)
    b = b.subset(np.nonzero(b.kind == W.PUT)[0][:8])
    try:
        api.debug_set_split_mode(1)
        api.debug_set_light_split(light_split)
        got, rc = api.price_american_tc_batch_host(b, N)
    finally:
        api.debug_set_split_mode(-1)
        api.debug_set_light_split(1)
    assert rc == 0
    assert_quotes(got, b, N)


def test_config5b_single_tree_split(api):
    """BASELINE config 5b shape at a size the oracle finishes quickly (N=1200),
    through the north-star single-option call (automatic split mode)."""
    r = W.config5b().row(0)
    N = 1200
    q = api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, r["k"], api.PUT)
    o = O.price_tc(_opt(r), N)
    assert q["status"] == 0 and close(q["ask"], o.ask, N) and close(q["bid"], o.bid, N), (q, o)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("N", [31, 64, 150])
def test_light_kernel_matches_full_kernel(api, mode, N):
    """Sellers and put buyers run on a light kernel by default (mode 1:
    amtc_light.cu; mode 2: the strip kernel's light variant); the full kernel
    must give the same prices and both must match the oracle.  N = 31 and 64
    leave ragged / exact last strips."""
    b = W.random_small(96, seed=6100 + N, k_max=0.05)
    try:
        api.debug_set_split_mode(0)
        api.debug_set_light_kernel(0)
        ref, rc0 = api.price_american_tc_batch_host(b, N)
        api.debug_set_light_kernel(mode)
        got, rc = api.price_american_tc_batch_host(b, N)
        st = api.tc_last_stats()
    finally:
        api.debug_set_light_kernel(1)
        api.debug_set_split_mode(-1)
    assert rc == 0 and rc0 == 0
    assert st["light_ms"] > 0.0  # the light kernel really ran
    np.testing.assert_allclose(got["ask"], ref["ask"], rtol=1e-12, atol=floor(N))
    np.testing.assert_allclose(got["bid"], ref["bid"], rtol=1e-12, atol=floor(N))
    assert_quotes(got, b, N)


def test_call_sellers_across_kh(api):
    """Call sellers grow 7-9 vertices at large k/h (oracle): below
    k/h = 4 they run on the light kernel, above on the full kernel; a light-
    kernel overflow would re-run the item on the full kernel.  All prices match."""
    b = W.random_small(64, seed=6200, k_max=0.05)
    b.kind[:] = W.CALL
    N = 400
    got, rc = api.price_american_tc_batch_host(b, N)
    assert rc == 0
    assert_quotes(got, b, N)


def test_config5b_full_size_golden(api):
    """BASELINE config 5b at full size (N=8000, k=0.005) through the north-star
    call (split mode), against the stored oracle value (scripts/make_oracle_refs.py)."""
    ref = json.load(open(os.path.join(GOLD, "oracle_config5b.json")))
    r = W.config5b().row(0)
    q = api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], ref["N"], r["k"], api.PUT)
    assert q["status"] == 0
    assert close(q["ask"], ref["ask"], ref["N"]) and close(q["bid"], ref["bid"], ref["N"]), (q, ref)


def test_capacity_retry_passes(api):
    """Shrunken arenas force heavy items through the retry passes (4x arenas per
    pass): same prices; with arenas too small for every pass, AMTC_ECAPACITY."""
    b = W.random_small(12, seed=99, k_max=0.0)
    b.kind[:] = 1
    b.k[:] = np.linspace(0.006, 0.02, 12)
    b.T[:] = 0.6
    b.sigma[:] = 0.3
    N = 400
    try:
        api.debug_set_split_mode(0)
        ref, rc0 = api.price_american_tc_batch_host(b, N)
        api.debug_set_arena_shift(9)
        got, rc = api.price_american_tc_batch_host(b, N)
        st = api.tc_last_stats()
        api.debug_set_arena_shift(16)
        bad, rc2 = api.price_american_tc_batch_host(b, N)
    finally:
        api.debug_set_arena_shift(0)
        api.debug_set_split_mode(-1)
    assert rc0 == 0 and rc == 0
    assert st["passes"] > 1 and st["retried_items"] > 0, st
    np.testing.assert_allclose(got["ask"], ref["ask"], rtol=1e-12, atol=floor(N))
    np.testing.assert_allclose(got["bid"], ref["bid"], rtol=1e-12, atol=floor(N))
    assert rc2 == 3 and np.any(bad["status"] == 3)  # AMTC_ECAPACITY
    assert np.all(np.isnan(bad["ask"][bad["status"] == 3]))


def test_fig9_curves(api):
    """the Fig. 9 workload as one batch at
    N=1000 -- parity with the oracle for all 63 points and the paper's ordering
    chain pi^b_k2 <= pi^b_k1 <= pi_k0 < pi^a_k1 < pi^a_k2 at every S0."""
    b = W.fig9()
    N = W.FIG9_N
    got, rc = api.price_american_tc_batch_host(b, N)
    assert rc == 0
    want = O.price_tc_many([_opt(b.row(i)) for i in range(len(b))], N)
    assert_quotes(got, b, N, want)
    a, bid = got["ask"].reshape(3, 21), got["bid"].reshape(3, 21)
    np.testing.assert_allclose(a[0], bid[0], rtol=1e-9)        # k = 0: ask = bid = CRR
    assert np.all(bid[2] <= bid[1] + 1e-10) and np.all(bid[1] <= bid[0] + 1e-10)
    assert np.all(a[0] < a[1]) and np.all(a[1] < a[2])


@pytest.mark.parametrize("N", [5, 60, 400])
def test_root_hedge(api, N):
    """the root hedges (positions at t = 0) through
    amtc_price_american_tc_hedge against the oracle's; at k = 0 they are the
    CRR delta and its negative (pinned in test_oracle_identities.py)."""
    b = W.random_small(16, seed=7000 + N, k_max=0.03)
    b.k[:4] = 0.0
    for i in range(len(b)):
        r = b.row(i)
        g = api.price_american_tc_hedge(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, r["k"], r["kind"], r["K2"])
        o = O.price_tc(_opt(r), N)
        assert g["status"] == o.status == 0
        assert close(g["ask"], o.ask, N) and close(g["bid"], o.bid, N), (i, g, o)
        for name, gy, oy in (("ask", g["hedge_ask"], o.hedge_ask), ("bid", g["hedge_bid"], o.hedge_bid)):
            assert abs(gy - oy) <= 1e-8 * (1.0 + abs(oy)), (i, name, gy, oy, r)


@pytest.mark.parametrize("N", [9, 120])
def test_european_and_cash_variants(api, N):
    """European (no exercise before N), cash-settled put /
    call and costs-at-t=0 variants through the batch flags, against the oracle's
    variants (pinned to the closed-form sum and CRR at k = 0, and to the LP brute
    force for costs at t = 0)."""
    b = W.random_small(40, seed=8000 + N, k_max=0.03)
    rng = np.random.default_rng(N)
    flags = rng.integers(0, 8, len(b)).astype(np.uint32)  # EUROPEAN | CASH | COST_AT_T0
    flags[b.kind == 2] &= 5  # cash settlement is for puts and calls (bull spreads are cash already)
    cols = {f: getattr(b, f) for f in W.Batch.fields()}
    cols["flags"] = flags
    got, rc = api.price_american_tc_batch_host(cols, N)
    assert rc == 0
    want = []
    for i in range(len(b)):
        r = b.row(i)
        want.append(O.price_tc(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], r["k"], r["kind"], r["K2"],
                                        american=not (flags[i] & 1), cash=bool(flags[i] & 2),
                                        cost_t0=bool(flags[i] & 4)), N))
    assert_quotes(got, b, N, want)
    # k = 0 CRR kernels: European / cash on the batch CRR path and the single-tree path
    crr = api.price_crr_batch_host(cols, N)
    for i in range(len(b)):
        r = b.row(i)
        o = O.price_crr(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], 0.0, r["kind"], r["K2"],
                                 american=not (flags[i] & 1)), N)
        assert close(crr[i], o, N), (i, crr[i], o)
    # invalid: cash on a bull spread, unknown bit
    bad = dict(cols)
    bad["flags"] = np.where(b.kind == 2, 2, 16).astype(np.uint32)
    q, rc = api.price_american_tc_batch_host(bad, N)
    assert rc == 1 and np.all(q["status"] == 1)
