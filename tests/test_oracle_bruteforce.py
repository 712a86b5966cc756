"""Pin the oracle's TC recursion to the DEFINITION of the ask and bid:
superhedging LPs on the non-recombining path tree (tests/bruteforce.py), which
share no code with the oracle.  N <= 3 (the bid enumerates all stopping times)."""
import pytest

import bruteforce as B
import oracle as O

MARKETS = [
    # (S0, K, K2, T, sigma, R, kind)
    (100.0, 100.0, 0.0, 0.25, 0.2, 0.1, O.PUT),     # the paper's Ex. 5.1 put
    (100.0, 100.0, 0.0, 0.25, 0.2, 0.1, O.CALL),
    (100.0, 95.0, 105.0, 0.25, 0.2, 0.1, O.BULL),    # the paper's bull spread
    (100.0, 110.0, 0.0, 0.01, 0.1, 0.05, O.PUT),     # small h -> large k/h
    (100.0, 90.0, 0.0, 0.01, 0.1, 0.05, O.CALL),
    (100.0, 92.0, 108.0, 0.01, 0.15, 0.0, O.BULL),
]
KS = [0.0, 0.005, 0.02, 0.1]


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("m", range(len(MARKETS)))
def test_ask_bid_match_lp(m, k, N):
    S0, K, K2, T, sigma, R, kind = MARKETS[m]
    q = O.price_tc(O.Option(S0, K, T, sigma, R, k, kind, K2), N)
    assert q.status == 0
    ask = B.ask_lp(S0, K, T, sigma, R, k, N, kind, K2)
    bid = B.bid_enum(S0, K, T, sigma, R, k, N, kind, K2)
    scale = max(1.0, abs(ask))
    assert abs(q.ask - ask) <= 1e-8 * scale
    assert abs(q.bid - bid) <= 1e-8 * scale


@pytest.mark.slow
@pytest.mark.parametrize("k", [0.005, 0.05])
@pytest.mark.parametrize("m", [0, 1, 2, 4])
def test_ask_bid_match_lp_n3(m, k):
    S0, K, K2, T, sigma, R, kind = MARKETS[m]
    q = O.price_tc(O.Option(S0, K, T, sigma, R, k, kind, K2), 3)
    ask = B.ask_lp(S0, K, T, sigma, R, k, 3, kind, K2)
    bid = B.bid_enum(S0, K, T, sigma, R, k, 3, kind, K2)
    assert abs(q.ask - ask) <= 1e-8 * max(1.0, abs(ask))
    assert abs(q.bid - bid) <= 1e-8 * max(1.0, abs(ask))


def test_ask_lp_n4():
    """The ask LP alone is cheap at N = 4 (63 path nodes)."""
    for m in (0, 1, 4):
        S0, K, K2, T, sigma, R, kind = MARKETS[m]
        q = O.price_tc(O.Option(S0, K, T, sigma, R, 0.01, kind, K2), 4)
        ask = B.ask_lp(S0, K, T, sigma, R, 0.01, 4, kind, K2)
        assert abs(q.ask - ask) <= 1e-8 * max(1.0, abs(ask))


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("k", [0.005, 0.02, 0.1])
@pytest.mark.parametrize("m", [0, 1, 2, 3])
def test_cost_at_t0_matches_lp(m, k, N):
    """SURVEY 8(f) NEXT #3 variant: proportional costs also at t = 0 (quotes
    (1 +- k) S0 at the root instead of P:159's S0), pinned to the superhedging
    LP / stopping-time definition with the same root quotes."""
    S0, K, K2, T, sigma, R, kind = MARKETS[m]
    q = O.price_tc(O.Option(S0, K, T, sigma, R, k, kind, K2, cost_t0=True), N)
    assert q.status == 0
    ask = B.ask_lp(S0, K, T, sigma, R, k, N, kind, K2, cost_t0=True)
    bid = B.bid_enum(S0, K, T, sigma, R, k, N, kind, K2, cost_t0=True)
    scale = max(1.0, abs(ask))
    assert abs(q.ask - ask) <= 1e-7 * scale, (q.ask, ask)
    assert abs(q.bid - bid) <= 1e-7 * scale, (q.bid, bid)
    base = O.price_tc(O.Option(S0, K, T, sigma, R, k, kind, K2), N)
    assert q.ask >= base.ask - 1e-12 and q.bid <= base.bid + 1e-12  # costs at t=0 only widen the spread


@pytest.mark.parametrize("m,k", [(0, 0.005), (1, 0.05), (2, 0.05), (4, 0.005)])
def test_bid_milp_n4(m, k):
    """the bid at N = 4 against the stopping-time MILP (one binary
    stop decision per path node, 63 of them; 458,330 stopping times are never
    enumerated).  P:92 defines the bid as the buyer's maximal borrowing."""
    S0, K, K2, T, sigma, R, kind = MARKETS[m]
    q = O.price_tc(O.Option(S0, K, T, sigma, R, k, kind, K2), 4)
    bid = B.bid_milp(S0, K, T, sigma, R, k, 4, kind, K2)
    assert abs(q.bid - bid) <= 1e-8 * max(1.0, abs(q.ask)), (q.bid, bid)


@pytest.mark.parametrize("N", [1, 2])
def test_bid_milp_equals_enumeration(N):
    """The MILP encoding of tau agrees with the exhaustive enumeration where both run."""
    for m in (0, 1, 2):
        S0, K, K2, T, sigma, R, kind = MARKETS[m]
        a = B.bid_milp(S0, K, T, sigma, R, 0.02, N, kind, K2)
        b = B.bid_enum(S0, K, T, sigma, R, 0.02, N, kind, K2)
        assert abs(a - b) <= 1e-8 * max(1.0, abs(b))
