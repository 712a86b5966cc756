"""Thin ctypes binding of include/amtc.h (argument marshalling only).

Every computation happens inside libamtc.so (CUDA, sm_100a, fp64).  PyTorch is
used only for device memory and streams.  There is no CPU fallback: loading
fails loudly when the library is missing.

Names follow the C-ABI: ``price_american_tc``, ``price_american_tc_batch``,
``price_american_tc_batch_host``, ``price_crr_batch``, ``price_crr_batch_host``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libamtc.so")

PUT, CALL, BULL = 0, 1, 2
EUROPEAN, CASH, COST_AT_T0 = 1, 2, 4  # payoff flags (AMTC_EUROPEAN, AMTC_CASH, AMTC_COST_AT_T0)
STATUS = {0: "OK", 1: "EINVAL", 2: "EARBITRAGE", 3: "ECAPACITY", 4: "EUNBOUNDED", 5: "ECUDA", 6: "ENCCL"}


class Params(C.Structure):
    _fields_ = [("S0", C.c_double), ("T", C.c_double), ("sigma", C.c_double), ("R", C.c_double)]


class Payoff(C.Structure):
    _fields_ = [("kind", C.c_int32), ("flags", C.c_uint32), ("K", C.c_double), ("K2", C.c_double)]


class Quote(C.Structure):
    _fields_ = [("ask", C.c_double), ("bid", C.c_double), ("status", C.c_int32), ("max_bp", C.c_int32)]


class BatchSoA(C.Structure):
    _fields_ = [("S0", C.c_void_p), ("K", C.c_void_p), ("K2", C.c_void_p), ("T", C.c_void_p),
                ("sigma", C.c_void_p), ("R", C.c_void_p), ("k", C.c_void_p), ("kind", C.c_void_p),
                ("flags", C.c_void_p)]


class TcStats(C.Structure):
    _fields_ = [("vertex_sum", C.c_int64), ("passes", C.c_int32), ("pad", C.c_int32),
                ("retried_items", C.c_int64), ("solve_ms", C.c_double), ("full_ms", C.c_double),
                ("light_ms", C.c_double)]


class Band(C.Structure):
    _fields_ = [("t_top", C.c_int32), ("Dp", C.c_int32), ("own_lo", C.c_int64), ("own_hi", C.c_int64),
                ("new_lo", C.c_int64), ("new_hi", C.c_int64), ("win_lo", C.c_int64), ("win_hi", C.c_int64),
                ("cap", C.c_int64)]


QUOTE_DTYPE = np.dtype([("ask", "<f8"), ("bid", "<f8"), ("status", "<i4"), ("max_bp", "<i4")])
assert QUOTE_DTYPE.itemsize == C.sizeof(Quote) == 24

EXPORTS = ["amtc_price_american_tc", "amtc_price_american_tc_batch", "amtc_price_american_tc_batch_host",
           "amtc_price_crr_batch", "amtc_price_crr_batch_host", "amtc_strerror", "amtc_last_error",
           "amtc_launch_count", "amtc_tc_last_stats", "amtc_debug_set_heavy_threshold",
           "amtc_price_crr_tree", "amtc_comm_unique_id", "amtc_comm_init", "amtc_comm_destroy",
           "amtc_price_tree_sharded", "amtc_debug_set_split_mode", "amtc_debug_set_light_kernel", "amtc_debug_set_full_kernel", "amtc_debug_set_light_split", "amtc_debug_full_profile",
           "amtc_debug_set_arena_shift", "amtc_tree_shard_plan", "amtc_price_american_tc_hedge",
           "amtc_batch_shard_plan", "amtc_tree_band_plan", "amtc_debug_set_tree_shape"]

_lib = None


def lib():
    """Load libamtc.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.amtc_price_american_tc.restype = Quote
        L.amtc_price_american_tc.argtypes = [C.POINTER(Params), C.c_int32, C.POINTER(Payoff), C.c_double]
        for name in ("amtc_price_american_tc_batch", "amtc_price_american_tc_batch_host"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(BatchSoA), C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        for name in ("amtc_price_crr_batch", "amtc_price_crr_batch_host"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(BatchSoA), C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.amtc_strerror.restype = C.c_char_p
        L.amtc_strerror.argtypes = [C.c_int]
        L.amtc_last_error.restype = C.c_char_p
        L.amtc_launch_count.restype = C.c_int64
        L.amtc_tc_last_stats.restype = C.c_int
        L.amtc_tc_last_stats.argtypes = [C.POINTER(TcStats)]
        L.amtc_price_crr_tree.argtypes = [C.POINTER(Params), C.c_int32, C.POINTER(Payoff),
                                          C.POINTER(C.c_double), C.c_void_p]
        L.amtc_comm_unique_id.argtypes = [C.c_char_p]
        L.amtc_comm_init.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.amtc_comm_destroy.argtypes = [C.c_void_p]
        L.amtc_price_tree_sharded.argtypes = [C.POINTER(Params), C.c_int32, C.POINTER(Payoff), C.c_double,
                                              C.c_void_p, C.c_int, C.c_int, C.POINTER(Quote), C.c_void_p]
        L.amtc_tree_shard_plan.argtypes = [C.c_int32, C.c_int, C.POINTER(C.c_int32)]
        L.amtc_tree_band_plan.argtypes = [C.c_int32, C.c_int, C.c_int, C.c_int32, C.c_int32, C.c_int64,
                                          C.POINTER(Band), C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
        L.amtc_batch_shard_plan.argtypes = [C.POINTER(BatchSoA), C.c_int64, C.c_int32, C.c_int, C.c_void_p,
                                            C.c_void_p]
        L.amtc_price_american_tc_hedge.argtypes = [C.POINTER(Params), C.c_int32, C.POINTER(Payoff), C.c_double,
                                                   C.POINTER(Quote), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.amtc_debug_set_tree_shape.restype = None
        L.amtc_debug_set_tree_shape.argtypes = [C.c_int]
        L.amtc_debug_set_arena_shift.restype = None
        L.amtc_debug_set_arena_shift.argtypes = [C.c_int]
        L.amtc_debug_full_profile.argtypes = [C.c_void_p, C.c_int]
        L.amtc_debug_set_full_kernel.restype = None
        L.amtc_debug_set_full_kernel.argtypes = [C.c_int]
        L.amtc_debug_set_light_split.restype = None
        L.amtc_debug_set_light_split.argtypes = [C.c_int]
        L.amtc_debug_set_light_kernel.restype = None
        L.amtc_debug_set_light_kernel.argtypes = [C.c_int]
        L.amtc_debug_set_split_mode.restype = None
        L.amtc_debug_set_split_mode.argtypes = [C.c_int]
        L.amtc_debug_set_heavy_threshold.restype = None
        L.amtc_debug_set_heavy_threshold.argtypes = [C.c_int]
        _lib = L
    return _lib


def _check(rc: int, allow_option_status: bool = True) -> int:
    if rc in (5, 6) or (rc != 0 and not allow_option_status):
        msg = lib().amtc_last_error().decode()
        raise RuntimeError(f"amtc error {STATUS.get(rc, rc)}: {msg}")
    return rc


def strerror(status: int) -> str:
    return lib().amtc_strerror(status).decode()


def launch_count() -> int:
    return int(lib().amtc_launch_count())


def debug_set_heavy_threshold(tl: int) -> None:
    """Testing hook: route node updates whose children hold > tl vertices to the
    warp-cooperative path (tl <= 0: default)."""
    lib().amtc_debug_set_heavy_threshold(int(tl))


def debug_set_tree_shape(shape: int) -> None:
    """Testing hook: k=0 single-tree sweep -- 0 auto (wavefront), 1 one launch per band,
    2..5 wavefront shapes (M, D) = (16, 256), (8, 128), (12, 128), (8, 64)."""
    lib().amtc_debug_set_tree_shape(int(shape))


def debug_set_split_mode(mode: int) -> None:
    """Testing hook: -1 automatic, 0 whole-tree warps only, 1 strip-split mode when it fits."""
    lib().amtc_debug_set_split_mode(int(mode))


def debug_set_light_kernel(on: bool) -> None:
    """Testing hook: run sellers / put buyers on the light kernel variant (default on)."""
    lib().amtc_debug_set_light_kernel(int(on))  # 0 off, 1 amtc_light.cu (default), 2 strip-kernel variant


def debug_set_full_kernel(which: int) -> None:
    """Testing hook: 1 the full solver of amtc_full.cu, 0 the strip kernel (default)."""
    lib().amtc_debug_set_full_kernel(int(which))


def debug_set_light_split(on: bool) -> None:
    """Testing hook: split mode of the light kernel for batches of light trees (default on)."""
    lib().amtc_debug_set_light_split(int(on))


def debug_full_profile(reset: bool = True):
    """Developer hook: the full solver's phase counters (None unless built with -DAMTC_F_PROF=1)."""
    out = np.zeros(8, dtype=np.uint64)
    rc = lib().amtc_debug_full_profile(out.ctypes.data, int(reset))
    if rc:
        return None
    keys = ("heavy_cycles", "wait_cycles", "idle_cycles", "total_cycles", "served", "post_levels", "tier2_cycles", "r7")
    return {k: int(v) for k, v in zip(keys, out)}


def debug_set_arena_shift(shift: int) -> None:
    """Testing hook: shrink the solver's arenas by 2**shift (0 restores them)."""
    lib().amtc_debug_set_arena_shift(int(shift))


def tc_last_stats() -> dict:
    s = TcStats()
    lib().amtc_tc_last_stats(C.byref(s))
    return {"vertex_sum": s.vertex_sum, "passes": s.passes, "retried_items": s.retried_items,
            "solve_ms": s.solve_ms, "full_ms": s.full_ms, "light_ms": s.light_ms}


# ---------------------------------------------------------------------------
# single option (north star)
# ---------------------------------------------------------------------------

def price_american_tc(S0: float, K: float, T: float, sigma: float, R: float, N: int, k: float,
                      kind: int = PUT, K2: float = 0.0, flags: int = 0) -> dict:
    """Ask and bid of one option under proportional costs k (flags: EUROPEAN | CASH)."""
    p = Params(S0, T, sigma, R)
    y = Payoff(kind, flags, K, K2)
    q = lib().amtc_price_american_tc(C.byref(p), N, C.byref(y), k)
    return {"ask": q.ask, "bid": q.bid, "status": q.status, "max_bp": q.max_bp}


# ---------------------------------------------------------------------------
# batches
# ---------------------------------------------------------------------------

_FIELDS = ("S0", "K", "K2", "T", "sigma", "R", "k", "kind", "flags")


def _soa_from_torch(cols: dict) -> BatchSoA:
    ptr = {f: (cols[f].data_ptr() if cols.get(f) is not None else None) for f in _FIELDS}
    return BatchSoA(**ptr)


def _soa_from_numpy(cols: dict):
    keep = {}
    for f in _FIELDS:
        a = cols.get(f)
        if a is None:
            keep[f] = None
            continue
        dt = np.int32 if f == "kind" else (np.uint32 if f == "flags" else np.float64)
        keep[f] = np.ascontiguousarray(a, dtype=dt)
    soa = BatchSoA(**{f: (keep[f].ctypes.data if keep[f] is not None else None) for f in _FIELDS})
    return soa, keep


def device_batch(batch, device="cuda"):
    """Copy a workloads.Batch (numpy SoA) to device tensors (dict)."""
    import torch
    out = {}
    for f in _FIELDS:
        a = getattr(batch, f, None)
        if a is None:
            continue
        out[f] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return out


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def price_american_tc_batch(cols: dict, N: int, out=None, stream=None):
    """Device batch: cols = dict of CUDA tensors (float64 / int32 'kind').
    Returns (quotes uint8 tensor viewable as QUOTE_DTYPE, status)."""
    import torch
    n = int(cols["S0"].numel())
    if out is None:
        out = torch.empty(n * 24, dtype=torch.uint8, device=cols["S0"].device)
    soa = _soa_from_torch(cols)
    rc = lib().amtc_price_american_tc_batch(C.byref(soa), n, N, C.c_void_p(out.data_ptr()),
                                            _stream_handle(stream))
    return out, _check(rc)


def quotes_to_numpy(out) -> np.ndarray:
    return out.cpu().numpy().view(QUOTE_DTYPE)


def price_american_tc_batch_host(batch, N: int, stream=None) -> tuple[np.ndarray, int]:
    """Host batch (numpy SoA, e.g. workloads.Batch); H2D/D2H inside the call."""
    cols = {f: getattr(batch, f, None) for f in _FIELDS} if not isinstance(batch, dict) else batch
    soa, keep = _soa_from_numpy(cols)
    n = len(keep["S0"])
    out = np.zeros(n, dtype=QUOTE_DTYPE)
    rc = lib().amtc_price_american_tc_batch_host(C.byref(soa), n, N, C.c_void_p(out.ctypes.data),
                                                 _stream_handle(stream))
    return out, _check(rc)


def price_crr_batch(cols: dict, N: int, out=None, stream=None):
    import torch
    n = int(cols["S0"].numel())
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=cols["S0"].device)
    soa = _soa_from_torch(cols)
    rc = lib().amtc_price_crr_batch(C.byref(soa), n, N, C.c_void_p(out.data_ptr()), _stream_handle(stream))
    _check(rc, allow_option_status=False)
    return out


def price_crr_batch_host(batch, N: int, stream=None) -> np.ndarray:
    cols = {f: getattr(batch, f, None) for f in _FIELDS} if not isinstance(batch, dict) else batch
    soa, keep = _soa_from_numpy(cols)
    n = len(keep["S0"])
    out = np.zeros(n, dtype=np.float64)
    rc = lib().amtc_price_crr_batch_host(C.byref(soa), n, N, C.c_void_p(out.ctypes.data),
                                         _stream_handle(stream))
    _check(rc, allow_option_status=False)
    return out


# ---------------------------------------------------------------------------
# one large tree (config 5): single GPU and sharded over an NCCL communicator
# ---------------------------------------------------------------------------

def price_crr_tree(S0: float, K: float, T: float, sigma: float, R: float, N: int, kind: int = PUT,
                   K2: float = 0.0, stream=None, flags: int = 0) -> float:
    """k = 0 CRR price of one (large) tree on the current device (flags: EUROPEAN | CASH)."""
    p = Params(S0, T, sigma, R)
    y = Payoff(kind, int(flags), K, K2)
    v = C.c_double()
    rc = lib().amtc_price_crr_tree(C.byref(p), N, C.byref(y), C.byref(v), _stream_handle(stream))
    if rc:
        raise ValueError(f"amtc_price_crr_tree: {STATUS.get(rc, rc)}")
    return v.value


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().amtc_comm_unique_id(buf)
    if rc:
        raise RuntimeError(f"amtc_comm_unique_id: {STATUS.get(rc, rc)}")
    return buf.raw


def comm_init(uid: bytes, nranks: int, rank: int) -> C.c_void_p:
    comm = C.c_void_p()
    rc = lib().amtc_comm_init(C.create_string_buffer(uid, 128), nranks, rank, C.byref(comm))
    if rc:
        raise RuntimeError(f"amtc_comm_init: {STATUS.get(rc, rc)}")
    return comm


def comm_destroy(comm) -> None:
    lib().amtc_comm_destroy(comm)


def comm_from_torch_dist(pg=None):
    """Create the library's NCCL communicator over the ranks of torch.distributed
    (the unique id travels through a broadcast_object_list)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(pg), dist.get_world_size(pg)
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=pg)
    return comm_init(obj[0], world, rank), rank, world


def price_tree_sharded(S0: float, K: float, T: float, sigma: float, R: float, N: int, k: float = 0.0,
                       kind: int = PUT, K2: float = 0.0, comm=None, rank: int = 0, nranks: int = 1,
                       stream=None) -> dict:
    """One tree sharded over the ranks of `comm` (every rank calls it)."""
    p = Params(S0, T, sigma, R)
    y = Payoff(kind, 0, K, K2)
    q = Quote()
    rc = lib().amtc_price_tree_sharded(C.byref(p), N, C.byref(y), k, comm, rank, nranks, C.byref(q),
                                       _stream_handle(stream))
    return {"ask": q.ask, "bid": q.bid, "status": q.status if rc == q.status else rc, "max_bp": q.max_bp}


def tree_shard_plan(N: int, nranks: int) -> list:
    """Strip partition of the sharded transaction-cost tree (host only)."""
    lo = (C.c_int32 * (nranks + 1))()
    rc = lib().amtc_tree_shard_plan(N, nranks, lo)
    if rc:
        raise ValueError(f"amtc_tree_shard_plan: {STATUS.get(rc, rc)}")
    return list(lo)


def tree_band_plan(N: int, nranks: int, rank: int, band: int = -1, D: int = 0, min_cols: int = 0):
    """Host-only exchange plan of one band of the k = 0 sharded tree, as rank
    `rank` executes it (amtc_tree_band_plan).  band = -1: the band count only.
    Returns (plan dict, send[nranks][2], recv[nranks][2]) or the count."""
    nb = C.c_int32(0)
    if band < 0:
        rc = lib().amtc_tree_band_plan(N, nranks, rank, -1, D, min_cols, None, None, None, C.byref(nb))
        if rc:
            raise ValueError(f"amtc_tree_band_plan: {STATUS.get(rc, rc)}")
        return nb.value
    b = Band()
    snd = np.zeros((nranks, 2), dtype=np.int64)
    rcv = np.zeros((nranks, 2), dtype=np.int64)
    rc = lib().amtc_tree_band_plan(N, nranks, rank, band, D, min_cols, C.byref(b), snd.ctypes.data,
                                   rcv.ctypes.data, C.byref(nb))
    if rc:
        raise ValueError(f"amtc_tree_band_plan: {STATUS.get(rc, rc)}")
    return {f: getattr(b, f) for f, _ in Band._fields_}, snd, rcv


def batch_shard_plan(batch, N: int, nranks: int):
    """Host-only deal of one option batch over nranks GPUs (amtc_batch_shard_plan:
    cost-sorted snake order, equal counts +-1).  Returns (rank_of[n] int32,
    rank_cost[nranks] float64)."""
    soa, keep = _soa_from_numpy({f: getattr(batch, f) for f in batch.fields()})
    n = len(batch)
    rank_of = np.empty(n, dtype=np.int32)
    cost = np.empty(nranks, dtype=np.float64)
    rc = lib().amtc_batch_shard_plan(C.byref(soa), n, N, nranks, rank_of.ctypes.data, cost.ctypes.data)
    if rc:
        raise ValueError(f"amtc_batch_shard_plan: {STATUS.get(rc, rc)}")
    return rank_of, cost


def price_american_tc_hedge(S0: float, K: float, T: float, sigma: float, R: float, N: int, k: float,
                            kind: int = PUT, K2: float = 0.0) -> dict:
    """Ask, bid and the root hedges (positions at t = 0) of one option."""
    p = Params(S0, T, sigma, R)
    y = Payoff(kind, 0, K, K2)
    q = Quote()
    ya, yb = C.c_double(), C.c_double()
    lib().amtc_price_american_tc_hedge(C.byref(p), N, C.byref(y), k, C.byref(q), C.byref(ya), C.byref(yb))
    return {"ask": q.ask, "bid": q.bid, "status": q.status, "max_bp": q.max_bp, "hedge_ask": ya.value,
            "hedge_bid": yb.value}
