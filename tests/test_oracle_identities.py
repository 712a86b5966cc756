"""Pins of the oracle by closed forms, exact identities and invariants.

  * k = 0: ask = bid = frictionless CRR American price (derived SURVEY A.1; the
    paper states pi^a_k0 = pi^b_k0 at P:364).  Two independent code paths:
    PWL recursion with the extra level N+1 vs scalar induction without it.
  * European CRR induction = closed-form binomial sum (log-space weights).
  * closed form -> Black-Scholes as N grows (textbook limit).
  * put-call parity of the European binomial prices (exact in the model).
  * American call without dividends = European call at k = 0.
  * ask non-decreasing and bid non-increasing in k; bid <= CRR <= ask;
    trivial-hedge bounds; Fig. 9 ordering chain.
"""
import math

import numpy as np
import pytest
from scipy.stats import norm

import oracle as O

PAPER_PUT = dict(S0=100.0, K=100.0, T=0.25, sigma=0.2, R=0.1)  # P:362 / P:389


@pytest.mark.parametrize("N", [1, 5, 20, 100, 400])
@pytest.mark.parametrize("kind,K,K2", [(O.PUT, 100.0, 0.0), (O.CALL, 100.0, 0.0), (O.BULL, 95.0, 105.0),
                                       (O.PUT, 85.0, 0.0), (O.CALL, 115.0, 0.0)])
def test_k0_equals_crr(N, kind, K, K2):
    o = O.Option(100.0, K, 0.25, 0.2, 0.1, 0.0, kind, K2)
    q = O.price_tc(o, N)
    crr = O.price_crr(o, N)
    assert q.status == 0
    assert q.ask == pytest.approx(crr, rel=1e-11, abs=1e-12)
    assert q.bid == pytest.approx(crr, rel=1e-11, abs=1e-12)


@pytest.mark.parametrize("N", [1, 7, 64, 500, 1500])
@pytest.mark.parametrize("kind", [O.PUT, O.CALL, O.BULL])
def test_european_induction_equals_closed_form(N, kind):
    o = O.Option(100.0, 105.0 if kind != O.BULL else 95.0, 0.7, 0.35, 0.04, 0.0, kind, 115.0, american=False)
    assert O.price_crr(o, N) == pytest.approx(O.price_euro_closed(o, N), rel=1e-11, abs=1e-13)


def _bs(S, K, T, sigma, R, call):
    d1 = (math.log(S / K) + (R + 0.5 * sigma ** 2) * T) / (sigma * math.sqrt(T))
    d2 = d1 - sigma * math.sqrt(T)
    if call:
        return S * norm.cdf(d1) - K * math.exp(-R * T) * norm.cdf(d2)
    return K * math.exp(-R * T) * norm.cdf(-d2) - S * norm.cdf(-d1)


@pytest.mark.parametrize("call", [False, True])
def test_closed_form_black_scholes_limit(call):
    o = O.Option(100.0, 100.0, 1.0, 0.3, 0.05, 0.0, O.CALL if call else O.PUT, american=False)
    bs = _bs(100.0, 100.0, 1.0, 0.3, 0.05, call)
    assert abs(O.price_euro_closed(o, 4000) - bs) < 5e-3  # O(1/N) binomial error


@pytest.mark.parametrize("N", [3, 100, 1024])
def test_put_call_parity(N):
    S0, K, T, sigma, R = 100.0, 93.0, 0.8, 0.25, 0.07
    c = O.price_euro_closed(O.Option(S0, K, T, sigma, R, 0.0, O.CALL, american=False), N)
    p = O.price_euro_closed(O.Option(S0, K, T, sigma, R, 0.0, O.PUT, american=False), N)
    assert c - p == pytest.approx(S0 - K * math.exp(-R * T), rel=1e-11)


@pytest.mark.parametrize("N", [10, 300, 1024])
@pytest.mark.parametrize("R", [0.0, 0.03, 0.1])
def test_american_call_equals_european(N, R):
    a = O.price_crr(O.Option(100.0, 97.0, 1.3, 0.4, R, 0.0, O.CALL), N)
    e = O.price_crr(O.Option(100.0, 97.0, 1.3, 0.4, R, 0.0, O.CALL, american=False), N)
    assert a == pytest.approx(e, rel=1e-12)


@pytest.mark.parametrize("kind,K,K2", [(O.PUT, 100.0, 0.0), (O.CALL, 100.0, 0.0), (O.BULL, 95.0, 105.0)])
def test_monotone_in_k_and_ordering(kind, K, K2):
    N = 150
    base = O.Option(100.0, K, 0.25, 0.2, 0.1, 0.0, kind, K2)
    crr = O.price_crr(base, N)
    prev = None
    for k in [0.0, 0.001, 0.0025, 0.005, 0.01, 0.02, 0.05]:
        q = O.price_tc(O.Option(100.0, K, 0.25, 0.2, 0.1, k, kind, K2), N)
        assert q.bid <= crr + 1e-12 <= q.ask + 2e-12
        if prev is not None:
            assert q.ask >= prev.ask - 1e-12
            assert q.bid <= prev.bid + 1e-12
        # trivial-hedge bounds
        xi0 = {O.PUT: K - 100.0, O.CALL: 100.0 - K, O.BULL: max(100.0 - K, 0) - max(100.0 - K2, 0)}[kind]
        assert q.bid >= max(xi0, 0.0) - 1e-12
        assert q.ask >= max(xi0, 0.0) - 1e-12
        bound = {O.PUT: K, O.CALL: 100.0, O.BULL: K2 - K}[kind]
        assert q.ask <= bound + 1e-12
        prev = q


def test_fig9_ordering_chain():
    """for S0 in [90, 110], pi^b_k2 <= pi^b_k1 <= pi_k0 < pi^a_k1 < pi^a_k2
    with k0 = 0, k1 = 0.25%, k2 = 0.5% (N unstated; reading A16 -> any N, here 200)."""
    N = 200
    for S0 in range(90, 111, 2):
        p = lambda k: O.price_tc(O.Option(float(S0), 100.0, 0.25, 0.2, 0.1, k, O.PUT), N)
        q0, q1, q2 = p(0.0), p(0.0025), p(0.005)
        assert q0.ask == pytest.approx(q0.bid, rel=1e-11)
        assert q2.bid <= q1.bid + 1e-12 <= q0.bid + 2e-12
        assert q0.ask < q1.ask < q2.ask


def test_invalid_inputs():
    bad = [
        O.Option(-1.0, 100.0, 1.0, 0.2, 0.05, 0.0),
        O.Option(100.0, 100.0, 0.0, 0.2, 0.05, 0.0),
        O.Option(100.0, 100.0, 1.0, 0.0, 0.05, 0.0),
        O.Option(100.0, 100.0, 1.0, 0.2, 0.05, 1.0),
        O.Option(100.0, 100.0, 1.0, 0.2, 0.05, -0.1),
        O.Option(100.0, 105.0, 1.0, 0.2, 0.05, 0.0, O.BULL, 95.0),
    ]
    for o in bad:
        assert O.price_tc(o, 10).status == O.EINVAL
    # arbitrage: r >= u  (R T/N >= sigma sqrt(T/N))
    assert O.price_tc(O.Option(100.0, 100.0, 1.0, 0.01, 0.5, 0.0), 4).status == O.EARBITRAGE


@pytest.mark.parametrize("kind,K,K2", [(O.PUT, 100.0, 0.0), (O.CALL, 95.0, 0.0), (O.BULL, 90.0, 110.0)])
@pytest.mark.parametrize("N", [3, 40])
def test_root_hedge_k0_is_crr_delta(kind, K, K2, N):
    """SURVEY 8(f) NEXT #2 pin (derived A.1): at k = 0 the seller's root hedge is
    the CRR delta (pi^u - pi^d) / (S0 (u - d)) of the level-1 CRR values, the
    buyer's its negative."""
    S0, T, sg, R = 100.0, 1.0, 0.3, 0.05
    q = O.price_tc(O.Option(S0, K, T, sg, R, 0.0, kind, K2), N)
    u = math.exp(sg * math.sqrt(T / N))
    d = 1.0 / u
    sub = lambda S: O.price_crr(O.Option(S, K, T * (N - 1) / N, sg, R, 0.0, kind, K2), N - 1)
    delta = (sub(S0 * u) - sub(S0 * d)) / (S0 * (u - d))
    assert q.hedge_ask == pytest.approx(delta, rel=1e-9, abs=1e-12)
    assert q.hedge_bid == pytest.approx(-delta, rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("kind,K,K2", [(O.PUT, 100.0, 0.0), (O.CALL, 95.0, 0.0), (O.BULL, 90.0, 110.0)])
@pytest.mark.parametrize("N", [7, 60])
def test_european_tc_k0_is_closed_form(kind, K, K2, N):
    """SURVEY 8(f) NEXT #3 pin: the European transaction-cost recursion (no
    exercise before N) at k = 0 equals the closed-form binomial sum (A.1 with the
    early max dropped); ask = bid."""
    o = O.Option(100.0, K, 0.9, 0.25, 0.04, 0.0, kind, K2, american=False)
    q = O.price_tc(o, N)
    ref = O.price_euro_closed(O.Option(100.0, K, 0.9, 0.25, 0.04, 0.0, kind, K2), N)
    assert q.ask == pytest.approx(ref, rel=1e-10) and q.bid == pytest.approx(ref, rel=1e-10)


@pytest.mark.parametrize("kind", [O.PUT, O.CALL])
def test_cash_settled_k0_is_crr(kind):
    """NEXT #3 pin: at k = 0 settlement does not matter (A.1): cash = CRR price."""
    for N in (5, 80):
        o = O.Option(100.0, 104.0, 0.7, 0.3, 0.05, 0.0, kind, cash=True)
        q = O.price_tc(o, N)
        ref = O.price_crr(O.Option(100.0, 104.0, 0.7, 0.3, 0.05, 0.0, kind), N)
        assert q.ask == pytest.approx(ref, rel=1e-10) and q.bid == pytest.approx(ref, rel=1e-10)


@pytest.mark.parametrize("kind", [O.PUT, O.CALL])
def test_european_below_american_with_costs(kind):
    """NEXT #3 invariant: fewer exercise rights -- the European ask is at most
    the American ask and the European bid at most the American bid (k > 0)."""
    for k in (0.005, 0.02):
        am = O.price_tc(O.Option(100.0, 100.0, 1.0, 0.2, 0.05, k, kind), 60)
        eu = O.price_tc(O.Option(100.0, 100.0, 1.0, 0.2, 0.05, k, kind, american=False), 60)
        assert eu.ask <= am.ask + 1e-12 and eu.bid <= am.bid + 1e-12
        assert eu.bid <= eu.ask


# --- SURVEY 8(c2) step 9 instrumentation: cost-model counters and level stats ---

def test_level_stats_consistent_with_quote():
    """The per-level kink statistics account for every node t <= N exactly once
    and agree with the quote's own max / sum of kinks."""
    N = 60
    o = O.Option(100.0, 105.0, 0.5, 0.15, 0.05, 0.02, O.CALL)
    L = O.new_level_stats(N)
    q = O.price_tc(o, N, level_stats=L)
    nodes = L[:, :, 2:].sum(axis=2)
    assert (nodes == np.arange(1, N + 2)[None, :]).all()
    assert L[0, :, 1].sum() == q.sum_kinks_ask and L[1, :, 1].sum() == q.sum_kinks_bid
    assert L[0, :, 0].max() == q.max_kinks_ask and L[1, :, 0].max() == q.max_kinks_bid
    # accumulation: a second call adds the same counts again
    q2 = O.price_tc(o, N, level_stats=L)
    assert L[0, :, 1].sum() == 2 * q.sum_kinks_ask and q2.fp64_ops == q.fp64_ops


def test_cost_model_counts():
    """fp64_ops applies the SURVEY 8(d) weights to the counted events; the seller
    (convex, A.3) never takes a non-convex restriction step, so at k=0 (all
    functions lines, A.1) every restriction step is convex."""
    N = 40
    q = O.price_tc(O.Option(100.0, 100.0, 1.0, 0.2, 0.05, 0.0, O.PUT), N)
    assert q.fp64_ops == (3 * q.merge_visits + 4 * q.crossings + 2 * q.restrict_cvx
                          + 4 * q.restrict_ncvx + 2 * q.scale_visits)
    assert q.restrict_ncvx == 0
    assert q.fp64_ops_ask + q.fp64_ops_bid == q.fp64_ops
    nodes = (N + 1) * (N + 2) // 2
    # every node update restricts both parties' w/r: two scan passes over >= 1 vertex
    assert q.restrict_cvx >= 2 * 2 * nodes and q.scale_visits >= 2 * nodes
    qk = O.price_tc(O.Option(100.0, 100.0, 1.0, 0.2, 0.05, 0.02, O.CALL), N)
    assert qk.restrict_ncvx > 0  # the buyer's z is non-convex


def test_kink_bins_cover_counts():
    for c in list(range(0, 300)) + [1000, 2047, 2048, 3001, 65535, 100000]:
        lo_bins = [b for b in range(240) if O.kink_bin_hi(b) >= c]
        b = lo_bins[0]
        assert O.kink_bin_hi(b) >= c and (b == 0 or O.kink_bin_hi(b - 1) < c)
