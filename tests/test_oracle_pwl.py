"""Pins of the oracle's PWL algebra by brute force on grids (SPEC's property suite,
S:115-117): pointwise max/min, slope restriction = infimal convolution with the
cost cone (reading R7), evaluated by brute-force minimisation over a fine y'
grid plus all vertices; invariants: slope bounds, result <= input,
idempotence, Unbounded detection."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O


def random_pwl(rng, n, convex=False, slope_lo=-3.0, slope_hi=3.0):
    x = np.sort(rng.uniform(-3, 3, n))
    x = np.unique(np.round(x, 6))
    s = rng.uniform(slope_lo, slope_hi, len(x) + 1)
    if convex:
        s = np.sort(s)
    f = np.empty(len(x))
    f[0] = rng.uniform(-2, 2)
    for i in range(1, len(x)):
        f[i] = f[i - 1] + s[i] * (x[i] - x[i - 1])
    return (x, f, float(s[0]), float(s[-1]))


def brute_eval(p, y):
    return O.pwl_eval(p, y)


def brute_restrict(p, lo, hi, ys):
    """v(y) = min over y' of f(y') + lo (y - y') [y' >= y] / hi (y - y') [y' <= y]."""
    x = p[0]
    grid = np.unique(np.concatenate([np.linspace(-12, 12, 24001), x, ys]))
    fg = O.pwl_eval(p, grid)
    out = []
    for y in ys:
        d = y - grid
        c = np.where(d <= 0, lo * d, hi * d)
        out.append(np.min(fg + c))
    return np.array(out)


seeds = st.integers(min_value=0, max_value=2**31 - 1)


@settings(max_examples=150, deadline=None)
@given(seeds, st.integers(1, 8), st.integers(1, 8))
def test_max_min_pointwise(seed, n1, n2):
    rng = np.random.default_rng(seed)
    f = random_pwl(rng, n1)
    g = random_pwl(rng, n2)
    ys = np.concatenate([rng.uniform(-8, 8, 300), f[0], g[0]])
    for op, fn in (("max", np.maximum), ("min", np.minimum)):
        h = O.pwl_op(op, f, g)
        want = fn(O.pwl_eval(f, ys), O.pwl_eval(g, ys))
        got = O.pwl_eval(h, ys)
        assert np.all(np.abs(got - want) <= 1e-9 * (1 + np.abs(want)))
        assert np.all(np.diff(h[0]) > 0)


@settings(max_examples=120, deadline=None)
@given(seeds, st.integers(1, 8), st.booleans())
def test_restrict_is_infimal_convolution(seed, n, convex):
    rng = np.random.default_rng(seed)
    lo = -float(rng.uniform(1.5, 2.5))
    hi = -float(rng.uniform(0.2, 1.0))
    # tails steeper than the interval on both sides keep the restriction finite
    f = random_pwl(rng, n, convex=convex, slope_lo=-4.0, slope_hi=1.0)
    f = (f[0], f[1], -4.0 + float(rng.uniform(-1, 0)), 1.0 + float(rng.uniform(0, 1)))
    f = O.pwl_op("canon", f)  # tails changed: rebuild values consistently below
    v = O.pwl_op("restrict", f, a=lo, b=hi)
    ys = np.concatenate([rng.uniform(-6, 6, 60), f[0]])
    want = brute_restrict(f, lo, hi, ys)
    got = O.pwl_eval(v, ys)
    assert np.all(np.abs(got - want) <= 1e-6 * (1 + np.abs(want)))
    # slopes of v lie in [lo, hi]; v <= f; idempotent
    xs = v[0]
    slopes = np.concatenate([[v[2]], np.diff(v[1]) / np.diff(xs) if len(xs) > 1 else [], [v[3]]])
    assert np.all(slopes >= lo - 1e-9) and np.all(slopes <= hi + 1e-9)
    assert np.all(got <= O.pwl_eval(f, ys) + 1e-9)
    v2 = O.pwl_op("restrict", v, a=lo, b=hi)
    assert np.all(np.abs(O.pwl_eval(v2, ys) - got) <= 1e-10 * (1 + np.abs(got)))


def test_restrict_convex_is_clipping():
    """For convex f restriction = clip slopes and reconnect (the P:118 example)."""
    f = (np.array([-1.0, 0.5]), np.array([130.0, 100.0]), -144.0, -10.0)
    v = O.pwl_op("restrict", f, a=-120.0, b=-80.0)
    # slopes: -144 -> clipped to -120 left of -1; middle piece slope -20 -> hi
    np.testing.assert_allclose(O.pwl_eval(v, [-2.0, -1.0, 0.0]), [250.0, 130.0, 50.0])


def test_restrict_unbounded():
    line = (np.array([0.0]), np.array([0.0]), -150.0, -150.0)
    with pytest.raises(ArithmeticError):
        O.pwl_op("restrict", line, a=-120.0, b=-80.0)
    line = (np.array([0.0]), np.array([0.0]), -50.0, -50.0)
    with pytest.raises(ArithmeticError):
        O.pwl_op("restrict", line, a=-120.0, b=-80.0)


def test_canonicalize_drops_collinear():
    f = (np.array([-1.0, 0.0, 1.0]), np.array([2.0, 0.0, -2.0]), -2.0, -2.0)
    c = O.pwl_op("canon", f)
    assert len(c[0]) == 1
    np.testing.assert_allclose(O.pwl_eval(c, [-5.0, 5.0]), [10.0, -10.0])
