"""Seeded synthetic workloads (BASELINE.json configs 1-5).

This module holds NO arithmetic of the method: it only draws option parameters
from a seeded numpy PCG64 generator in a fixed order, exactly as SURVEY.md 8(d)
prescribes (K, T, sigma, R, [k], u_kind), and returns them as SoA numpy arrays.
Both the oracle tests and the CUDA path consume the same arrays; this is the
only module they share.  It imports nothing from the rest of the package.

The paper measures on no public dataset (its workloads are the fixed put /
bull-spread examples of P:362); the batched configs 2 and 4 are
synthetic batches "shaped like the paper's workloads" (BASELINE.json).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PUT, CALL, BULL = 0, 1, 2
SEED_BASE = 0x11102477


@dataclass
class Batch:
    """Structure-of-arrays option batch (fp64 / int32), one entry per option."""
    S0: np.ndarray
    K: np.ndarray
    K2: np.ndarray
    T: np.ndarray
    sigma: np.ndarray
    R: np.ndarray
    k: np.ndarray
    kind: np.ndarray

    def __len__(self) -> int:
        return int(self.S0.shape[0])

    def subset(self, idx) -> "Batch":
        idx = np.asarray(idx)
        return Batch(*(np.ascontiguousarray(getattr(self, f)[idx]) for f in self.fields()))

    @staticmethod
    def fields():
        return ("S0", "K", "K2", "T", "sigma", "R", "k", "kind")

    def row(self, i: int) -> dict:
        return {f: (int(getattr(self, f)[i]) if f == "kind" else float(getattr(self, f)[i]))
                for f in self.fields()}


def soa_sha256(b: Batch) -> str:
    """SHA-256 of the batch's SoA bytes (fields in Batch.fields() order,
    little-endian fp64 / int32): the key of the cached oracle reference files."""
    import hashlib
    h = hashlib.sha256()
    for f in Batch.fields():
        a = getattr(b, f)
        h.update(np.ascontiguousarray(a, dtype=a.dtype.newbyteorder("<")).tobytes())
    return h.hexdigest()


def concat(batches) -> Batch:
    """Concatenate batches (e.g. the single-tree points of one N)."""
    return Batch(*(np.concatenate([getattr(b, f) for b in batches]) for f in Batch.fields()))


def _batch(S0, K, K2, T, sigma, R, k, kind) -> Batch:
    n = len(K)
    f = lambda a: np.array(np.broadcast_to(np.asarray(a, dtype=np.float64), (n,)), copy=True)
    return Batch(f(S0), f(K), f(K2), f(T), f(sigma), f(R), f(k),
                 np.array(np.broadcast_to(np.asarray(kind, dtype=np.int32), (n,)), copy=True))


def config1(k: float = 0.005) -> Batch:
    """Config 1: single American put S0=K=100, T=0.25, sigma=0.2, R=0.1, N=100
    (the paper's Example 5.1 put)."""
    return _batch(100.0, [100.0], 0.0, 0.25, 0.2, 0.1, k, PUT)


CONFIG1_N = 100


def config2(n: int = 65536, seed: int = SEED_BASE + 2) -> Batch:
    """Config 2: zero-cost batched American puts/calls, N=1024."""
    g = np.random.Generator(np.random.PCG64(seed))
    K = g.uniform(80.0, 120.0, n)
    T = g.uniform(0.1, 2.0, n)
    sigma = g.uniform(0.1, 0.6, n)
    R = g.uniform(0.0, 0.1, n)
    u_kind = g.uniform(0.0, 1.0, n)
    kind = np.where(u_kind < 0.5, PUT, CALL)
    return _batch(100.0, K, 0.0, T, sigma, R, 0.0, kind)


CONFIG2_N = 1024


def config3():
    """Config 3: single-tree sweep, put and call, S0=K=100, T=1, sigma=0.2,
    R=0.05, k in {0, .0025, .005, .01, .02} x N in {250, 500, 1000, 1500, 2000}.
    Returns a list of (Batch of one option, N)."""
    out = []
    for kind in (PUT, CALL):
        for k in (0.0, 0.0025, 0.005, 0.01, 0.02):
            for N in (250, 500, 1000, 1500, 2000):
                out.append((_batch(100.0, [100.0], 0.0, 1.0, 0.2, 0.05, k, kind), N))
    return out


def config4(n: int = 16384, seed: int = SEED_BASE + 4) -> Batch:
    """Config 4: batched transaction-cost pricing, N=1500.  Per option:
    K~U[80,120], T~U[.25,1], sigma~U[.1,.5], R~U[0,.08], k~U[0,.02];
    kind u<.45 put, <.90 call, else bull spread (K1=K-10, K2=K+10, cash)."""
    g = np.random.Generator(np.random.PCG64(seed))
    K = g.uniform(80.0, 120.0, n)
    T = g.uniform(0.25, 1.0, n)
    sigma = g.uniform(0.1, 0.5, n)
    R = g.uniform(0.0, 0.08, n)
    k = g.uniform(0.0, 0.02, n)
    u_kind = g.uniform(0.0, 1.0, n)
    kind = np.where(u_kind < 0.45, PUT, np.where(u_kind < 0.90, CALL, BULL)).astype(np.int32)
    K1 = np.where(kind == BULL, K - 10.0, K)
    K2 = np.where(kind == BULL, K + 10.0, 0.0)
    return _batch(100.0, K1, K2, T, sigma, R, k, kind)


CONFIG4_N = 1500


def config5a() -> Batch:
    """Config 5a: American put S0=K=100, T=1, sigma=0.3, R=0.05, k=0, N=100000."""
    return _batch(100.0, [100.0], 0.0, 1.0, 0.3, 0.05, 0.0, PUT)


def config5b() -> Batch:
    """Config 5b: the same put at k=0.005, N=8000."""
    return _batch(100.0, [100.0], 0.0, 1.0, 0.3, 0.05, 0.005, PUT)


CONFIG5A_N = 100000
CONFIG5B_N = 8000


def fig9(N_levels: int = 1000) -> Batch:
    """the paper's Fig. 9 price curves -- the
    Example 5.1 put (K=100, T=0.25, sigma=0.2, R=0.1) for S0 in {90, 91, ..., 110}
    and k in {0, 0.25%, 0.5%}, as one batch (k-major), to be priced at N=1000
    (reading A16)."""
    S0 = np.repeat(np.arange(90.0, 111.0)[None, :], 3, axis=0).ravel()
    k = np.repeat(np.array([0.0, 0.0025, 0.005]), 21)
    return _batch(S0, np.full(S0.shape, 100.0), 0.0, 0.25, 0.2, 0.1, k, PUT)


FIG9_N = 1000


def appendix_put() -> Batch:
    """Appendix workload: put K=S0=100, T=3, sigma=0.3, R=0.06."""
    return _batch(100.0, [100.0], 0.0, 3.0, 0.3, 0.06, 0.0, PUT)


def random_small(n: int, seed: int, k_max: float = 0.05) -> Batch:
    """Small random options for parity tests (all kinds, wide k/h range)."""
    g = np.random.Generator(np.random.PCG64(seed))
    K = g.uniform(80.0, 120.0, n)
    T = g.uniform(0.05, 1.0, n)
    sigma = g.uniform(0.05, 0.5, n)
    R = g.uniform(0.0, 0.08, n)
    k = g.uniform(0.0, k_max, n)
    u_kind = g.uniform(0.0, 1.0, n)
    kind = np.where(u_kind < 0.4, PUT, np.where(u_kind < 0.8, CALL, BULL)).astype(np.int32)
    K1 = np.where(kind == BULL, K - 10.0, K)
    K2 = np.where(kind == BULL, K + 10.0, 0.0)
    return _batch(100.0, K1, K2, T, sigma, R, k, kind)
