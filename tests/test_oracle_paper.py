"""Pins of the oracle against values the paper prints (tests/golden/paper_one_step.json).

P:n = /root/reference/PAPER.md line n (cited in the golden file)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_one_step.json")))


def kink_fn(d):
    """(x, f, sl, sr) of  value + (-sl)(y-kink)^- ... i.e. slope sl left, sr right."""
    return (np.array([d["kink"]]), np.array([d["value"]]), d["sl"], d["sr"])


def test_frictionless_one_step():
    """pi_t = max(30, 10.17) = 30 with u = 1.2, p = 0.9454 (so r = 1.18)."""
    g = GOLD["frictionless"]
    u = g["u"]
    d = 1.0 / u
    # the printed p fixes r through p = (r - d)/(u - d)
    r = d + g["p_printed"] * (u - d)
    assert abs(r - 1.18) < 5e-4
    r = 1.18  # reading A5: r = 1.18
    # one-step tree: sigma sqrt(T/N) = ln u, R T/N = ln r with T = N = 1
    opt = O.Option(S0=g["S"], K=g["K"], T=1.0, sigma=math.log(u), R=math.log(r), kind=O.PUT)
    assert O.price_crr(opt, 1) == pytest.approx(g["pi_t"], abs=1e-12)
    euro = O.Option(S0=g["S"], K=g["K"], T=1.0, sigma=math.log(u), R=math.log(r), kind=O.PUT, american=False)
    assert O.price_crr(euro, 1) == pytest.approx(g["discounted_expectation"], abs=5e-3)
    # the children values printed in the paper are the exercise values
    assert g["K"] - g["S"] * u == pytest.approx(g["child_values"][0], abs=1e-12)
    assert g["K"] - g["S"] * d == pytest.approx(g["child_values"][1], abs=5e-3)


@pytest.mark.parametrize("r", [1.001, 1.05, 1.18, 1.19])
def test_seller_one_step(r):
    """P:100-121, Eqs. (2)-(5).  The result is r-independent on (1, 1.2)
    (SURVEY A.5), so it is checked for several r including the read r = 1.18."""
    g = GOLD["seller"]
    zu = kink_fn(g["zu"])
    zd = kink_fn(dict(g["zd"], sr=-200.0 / 3.0))  # 66.67 = 200/3 printed to 2dp
    # w = max(z^u, z^d): kink at -1, slopes -144 / -66.67
    w = O.pwl_op("max", zu, zd)
    assert len(w[0]) == 1 and w[0][0] == pytest.approx(-1.0) and w[1][0] == pytest.approx(130.0)
    assert w[2] == pytest.approx(g["w"]["sl"]) and w[3] == pytest.approx(g["w"]["sr"], abs=5e-3)
    # restricted to [-120, -80]
    lo, hi = g["restrict_interval"]
    v = O.pwl_op("restrict", O.pwl_op("div", w, a=r), a=lo, b=hi)
    assert v[2] == pytest.approx(lo) and v[3] == pytest.approx(hi)
    Sa = (1 + g["k"]) * g["S"]
    Sb = (1 - g["k"]) * g["S"]
    assert (-Sa, -Sb) == pytest.approx((lo, hi))
    z = O.node_update(0, zu, zd, r, Sa, Sb, g["xi"], g["zeta"])
    ys = np.array([-3.0, -1.5, -1.0, -0.5, 0.0, 0.7, 2.0])
    want = np.where(ys < -1, g["z_pieces"]["left"][0] * ys + g["z_pieces"]["left"][1],
                    g["z_pieces"]["right"][0] * ys + g["z_pieces"]["right"][1])
    np.testing.assert_allclose(O.pwl_eval(z, ys), want, rtol=0, atol=1e-10)
    assert O.pwl_eval(z, 0.0)[0] == pytest.approx(g["ask"], abs=1e-12)


@pytest.mark.parametrize("r", [1.001, 1.05, 1.18, 1.19])
def test_buyer_one_step(r):
    """P:131-144, Eq. (7): z_t = min(u_t, v_t) = u_t; bid = -z_t(0) = 10."""
    g = GOLD["buyer"]
    zu = kink_fn(g["zu"])
    zd = kink_fn(dict(g["zd"], sr=-200.0 / 3.0))
    Sa = (1 + g["k"]) * g["S"]
    Sb = (1 - g["k"]) * g["S"]
    z = O.node_update(1, zu, zd, r, Sa, Sb, g["xi"], g["zeta"])
    ys = np.array([-2.0, 0.0, 0.5, 1.0, 1.5, 3.0])
    want = np.where(ys < 1, g["z_pieces"]["left"][0] * ys + g["z_pieces"]["left"][1],
                    g["z_pieces"]["right"][0] * ys + g["z_pieces"]["right"][1])
    np.testing.assert_allclose(O.pwl_eval(z, ys), want, rtol=0, atol=1e-10)
    assert -O.pwl_eval(z, 0.0)[0] == pytest.approx(g["bid"], abs=1e-12)


def test_appendix_put_13906():
    """the frictionless American put price 13.906 (N not stated, reading
    A16: Table III's range; at N = 10000 the CRR value rounds to 13.906)."""
    g = GOLD["appendix_put"]
    opt = O.Option(S0=g["S0"], K=g["K"], T=g["T"], sigma=g["sigma"], R=g["R"], kind=O.PUT)
    p = O.price_crr(opt, 10000)
    assert round(p, 3) == g["price_3dp"]


def test_calibration_formula_via_one_step_tree():
    """u = exp(sigma sqrt(T/N)), d = 1/u, r = exp(RT/N).  A one-step
    European call's CRR value (S0 u - K)^+ p / r fixes u, d, r jointly."""
    S0, K, T, sigma, R = 100.0, 100.0, 0.25, 0.2, 0.1
    N = 20
    u = math.exp(sigma * math.sqrt(T / N))
    assert u == pytest.approx(1.0226126, abs=5e-8)  # formula value
    assert math.exp(R * T / N) == pytest.approx(1.0012508, abs=5e-8)
    opt = O.Option(S0=S0, K=K, T=T / N, sigma=sigma, R=R, kind=O.CALL, american=False)
    d = 1 / u
    r = math.exp(R * T / N)
    p = (r - d) / (u - d)
    assert O.price_crr(opt, 1) == pytest.approx(p * (S0 * u - K) / r, rel=1e-13)
