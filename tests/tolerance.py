"""Parity tolerance of the CUDA path against the oracle (north star: 1e-9
relative in fp64) with DESIGN.md reading A19:

  |g - o| <= 1e-9 |o|             the north-star bound, or
  |g - o| <= FLOOR_C * N * eps * S0   the rounding floor (counted as floor_used).

A relative bound alone is undefined at o = 0 (deep out-of-the-money bids are
exactly 0 in the oracle) and unattainable for small prices: node-function
values are O(S0) and every one of the N levels rounds them, so two correct fp64
evaluation orders differ by O(N eps S0) in absolute terms, whatever the price.
FLOOR_C is set from the measured error histogram of the full config-4 and
config-2 batches against the oracle (profiles/r02_parity_error_hist.json,
DESIGN.md A19); tests report how many comparisons the floor decided."""
import numpy as np

RTOL = 1e-9
FLOOR_C = 4.0
EPS = float(np.finfo(np.float64).eps)


def floor(N, S0=100.0):
    return FLOOR_C * max(int(N), 1) * EPS * S0


def close(g, o, N, S0=100.0) -> bool:
    err = abs(g - o)
    return err <= RTOL * abs(o) or err <= floor(N, S0)


def check_arrays(g, o, N, S0=100.0):
    """Vectorised: returns (ok mask, number of entries decided by the floor)."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    S0 = np.broadcast_to(np.asarray(S0, dtype=np.float64), o.shape)
    err = np.abs(g - o)
    rel = err <= RTOL * np.abs(o)
    flo = err <= FLOOR_C * max(int(N), 1) * EPS * S0
    return rel | flo, int((flo & ~rel).sum())
