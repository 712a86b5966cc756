"""CPU oracle for the amtc hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
(``paper_1110_2477_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``amtc_oracle.c``, built with
``-O2 -ffp-contract=off``); this module only marshals arguments through
ctypes.  Every function cites the PAPER.md passage it follows in the C source.

Parity status of each oracle function:
  price_tc           pinned: paper one-step examples, k=0 identity
                     with CRR (derived A.1), LP/stopping-time brute force for
                     N <= 3 (definition of ask/bid), invariants.
  price_crr          pinned: paper one-step, 13.906,
                     closed-form European sum, American call = European call.
  price_euro_closed  pinned: Black-Scholes limit, put-call parity.
  pwl_op             pinned: grid brute force (max/min/restrict), paper Eq. 2-5.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "amtc_oracle.c")
_LIB = os.path.join(_HERE, "libamtc_oracle.so")

PUT, CALL, BULL = 0, 1, 2
OK, EINVAL, EARBITRAGE, EUNBOUNDED = 0, 1, 2, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Option(C.Structure):
    _fields_ = [("S0", C.c_double), ("K", C.c_double), ("K2", C.c_double), ("T", C.c_double),
                ("sigma", C.c_double), ("R", C.c_double), ("k", C.c_double),
                ("kind", C.c_int32), ("american", C.c_int32), ("cash", C.c_int32), ("cost_t0", C.c_int32)]


class _Quote(C.Structure):
    _fields_ = [("ask", C.c_double), ("bid", C.c_double), ("status", C.c_int32),
                ("max_kinks_ask", C.c_int32), ("max_kinks_bid", C.c_int32), ("pad", C.c_int32),
                ("sum_kinks_ask", C.c_int64), ("sum_kinks_bid", C.c_int64),
                ("crossings", C.c_int64), ("hedge_ask", C.c_double), ("hedge_bid", C.c_double),
                ("fp64_ops", C.c_int64), ("merge_visits", C.c_int64), ("restrict_cvx", C.c_int64),
                ("restrict_ncvx", C.c_int64), ("scale_visits", C.c_int64),
                ("fp64_ops_ask", C.c_int64), ("fp64_ops_bid", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        _lib.oracle_price_tc.argtypes = [C.POINTER(_Option), C.c_int, C.POINTER(_Quote), C.POINTER(C.c_int32)]
        _lib.oracle_price_tc_stats.argtypes = [C.POINTER(_Option), C.c_int, C.POINTER(_Quote),
                                               C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        _lib.oracle_kink_bin_hi.argtypes = [C.c_int]
        _lib.oracle_price_crr.argtypes = [C.POINTER(_Option), C.c_int, dp]
        _lib.oracle_price_euro_closed.argtypes = [C.POINTER(_Option), C.c_int, dp]
        _lib.oracle_pwl_op.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_double,
                                       C.c_int, dp, dp, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int, ip, dp, dp, dp, dp]
        _lib.oracle_pwl_eval.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, C.c_int, dp, dp]
        _lib.oracle_node_update.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_double,
                                            C.c_int, dp, dp, C.c_double, C.c_double,
                                            C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                            C.c_int, ip, dp, dp, dp, dp]
    return _lib


@dataclass
class Option:
    S0: float
    K: float
    T: float
    sigma: float
    R: float
    k: float = 0.0
    kind: int = PUT
    K2: float = 0.0
    american: bool = True
    cash: bool = False
    cost_t0: bool = False

    def _c(self) -> _Option:
        return _Option(self.S0, self.K, self.K2, self.T, self.sigma, self.R, self.k, self.kind,
                       1 if self.american else 0, 1 if self.cash else 0, 1 if self.cost_t0 else 0)


@dataclass
class Quote:
    ask: float
    bid: float
    status: int
    max_kinks_ask: int
    max_kinks_bid: int
    sum_kinks_ask: int
    sum_kinks_bid: int
    crossings: int
    hedge_ask: float = float("nan")
    hedge_bid: float = float("nan")
    # SURVEY 8(d) cost model, counted by the oracle (instrumentation only):
    # fp64_ops = 3 merge_visits + 4 crossings + 2 restrict_cvx + 4 restrict_ncvx
    #            + 2 scale_visits over every node t <= N, both parties
    fp64_ops: int = 0
    merge_visits: int = 0
    restrict_cvx: int = 0
    restrict_ncvx: int = 0
    scale_visits: int = 0
    fp64_ops_ask: int = 0  # fp64_ops of the seller's recursion (ask) ...
    fp64_ops_bid: int = 0  # ... and of the buyer's (bid)


def _quote(q) -> "Quote":
    return Quote(q.ask, q.bid, q.status, q.max_kinks_ask, q.max_kinks_bid, q.sum_kinks_ask,
                 q.sum_kinks_bid, q.crossings, q.hedge_ask, q.hedge_bid, q.fp64_ops,
                 q.merge_visits, q.restrict_cvx, q.restrict_ncvx, q.scale_visits, q.fp64_ops_ask,
                 q.fp64_ops_bid)


def lvl_stride() -> int:
    return lib().oracle_lvl_stride()


def new_level_stats(N: int) -> np.ndarray:
    """Accumulator for price_tc(..., level_stats=acc): int64 array of shape
    (2, N+1, stride); [p, t, 0] = max kinks on level t, [p, t, 1] = sum of kinks,
    [p, t, 2+b] = number of nodes in kink bin b (kink_bin_hi(b) = bin's top)."""
    return np.zeros((2, N + 1, lvl_stride()), dtype=np.int64)


def kink_bin_hi(b: int) -> int:
    return lib().oracle_kink_bin_hi(int(b))


def price_tc(opt: Option, N: int, kinks: bool = False, level_stats: np.ndarray | None = None):
    """Ask/bid under proportional costs (Sec. 3 + 4.1).  With kinks=True also
    returns the per-node kink counts, shape (N+1)(N+2)/2 x 2 (seller, buyer).
    level_stats (optional, from new_level_stats(N)) accumulates the per-level
    kink max / sum / histogram of this option into the caller's array."""
    q = _Quote()
    arr = None
    ptr = None
    if kinks:
        arr = np.zeros(((N + 1) * (N + 2) // 2, 2), dtype=np.int32)
        ptr = arr.ctypes.data_as(C.POINTER(C.c_int32))
    lptr = None
    if level_stats is not None:
        assert level_stats.dtype == np.int64 and level_stats.shape == (2, N + 1, lvl_stride())
        assert level_stats.flags.c_contiguous
        lptr = level_stats.ctypes.data_as(C.POINTER(C.c_int64))
    o = opt._c()
    lib().oracle_price_tc_stats(C.byref(o), N, C.byref(q), ptr, lptr)
    out = _quote(q)
    return (out, arr) if kinks else out


def price_crr(opt: Option, N: int) -> float:
    """Frictionless CRR price by backward induction."""
    v = C.c_double()
    o = opt._c()
    st = lib().oracle_price_crr(C.byref(o), N, C.byref(v))
    if st:
        raise ValueError(f"oracle_price_crr status {st}")
    return v.value


def price_euro_closed(opt: Option, N: int) -> float:
    """European CRR price, closed-form binomial sum."""
    v = C.c_double()
    o = opt._c()
    st = lib().oracle_price_euro_closed(C.byref(o), N, C.byref(v))
    if st:
        raise ValueError(f"oracle_price_euro_closed status {st}")
    return v.value


def price_tc_many(opts, N: int, threads: int | None = None):
    """price_tc over a list of options, parallel over options only (ctypes
    releases the GIL).  Returns a list of Quote."""
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda o: price_tc(o, N), opts))


def price_crr_many(opts, N: int, threads: int | None = None):
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda o: price_crr(o, N), opts))


# ---------------------------------------------------------------------------
# PWL functions as (x, f, sl, sr) tuples
# ---------------------------------------------------------------------------

def _arr(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _unpack(cap, n, x, f, sl, sr):
    return (x[: n.value].copy(), f[: n.value].copy(), sl.value, sr.value)


def pwl_op(op: str, p, q=None, a: float = 0.0, b: float = 0.0):
    """op in {'max','min','restrict','div','canon'}; p, q = (x, f, sl, sr)."""
    code = {"max": 0, "min": 1, "restrict": 2, "div": 3, "canon": 4}[op]
    x1, px1 = _arr(p[0])
    f1, pf1 = _arr(p[1])
    if q is None:
        q = p
    x2, px2 = _arr(q[0])
    f2, pf2 = _arr(q[1])
    cap = 4 * (len(x1) + len(x2)) + 16
    x, px = _arr(np.zeros(cap))
    f, pf = _arr(np.zeros(cap))
    n, sl, sr = C.c_int(), C.c_double(), C.c_double()
    st = lib().oracle_pwl_op(code, len(x1), px1, pf1, p[2], p[3], len(x2), px2, pf2, q[2], q[3],
                             a, b, cap, C.byref(n), px, pf, C.byref(sl), C.byref(sr))
    if st == EUNBOUNDED:
        raise ArithmeticError("Unbounded")
    if st:
        raise ValueError(f"oracle_pwl_op status {st}")
    return _unpack(cap, n, x, f, sl, sr)


def pwl_eval(p, y):
    x, px = _arr(p[0])
    f, pf = _arr(p[1])
    y, py = _arr(np.atleast_1d(y))
    out, po = _arr(np.zeros(len(y)))
    lib().oracle_pwl_eval(len(x), px, pf, p[2], p[3], len(y), py, po)
    return out


def node_update(party: int, zu, zd, r, Sa, Sb, xi, zeta):
    """One node of the seller (party 0) / buyer (party 1) recursion."""
    x1, px1 = _arr(zu[0])
    f1, pf1 = _arr(zu[1])
    x2, px2 = _arr(zd[0])
    f2, pf2 = _arr(zd[1])
    cap = 8 * (len(x1) + len(x2)) + 16
    x, px = _arr(np.zeros(cap))
    f, pf = _arr(np.zeros(cap))
    n, sl, sr = C.c_int(), C.c_double(), C.c_double()
    st = lib().oracle_node_update(party, len(x1), px1, pf1, zu[2], zu[3], len(x2), px2, pf2, zd[2], zd[3],
                                  r, Sa, Sb, xi, zeta, cap, C.byref(n), px, pf, C.byref(sl), C.byref(sr))
    if st:
        raise ValueError(f"oracle_node_update status {st}")
    return _unpack(cap, n, x, f, sl, sr)
