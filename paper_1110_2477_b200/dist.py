"""Batched multi-GPU pricing (SURVEY.md 8(e), row "Batched TC (config 4) and CRR
(config 2)"): ONE batch of independent options is dealt over the ranks by
estimated cost, every rank prices its share on its own GPU with no inter-GPU
traffic, and a single all-gather of the 24-byte quotes completes the batch
("The batched path instead splits options across the 8 B200s with no inter-GPU
traffic except a final gather", BASELINE.json north_star; the paper's per-round
load balancing, is the prior art for dealing by cost).

The deal is the library's host-only `amtc_batch_shard_plan` (cost-sorted snake
order, equal counts +-1); the gather is `torch.distributed.all_gather_into_tensor`
over the caller's process group (NCCL on GPUs; gloo in the CPU tests, where a
test-supplied pricer stands in for the GPU).  Pure plumbing: no arithmetic of the
method lives here.
"""
from __future__ import annotations

import numpy as np

from . import api

QUOTE_BYTES = 24


def plan(batch, N: int, nranks: int):
    """(rank_of[n], rank_cost[nranks]) from the library's host-only deal."""
    return api.batch_shard_plan(batch, N, nranks)


def local_indices(rank_of: np.ndarray, rank: int) -> np.ndarray:
    """Batch positions priced by `rank`, in batch order."""
    return np.nonzero(rank_of == rank)[0]


def gather_quotes(local, rank_of: np.ndarray, rank: int, nranks: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's quotes and scatter them back to batch order.

    local: this rank's quotes in local_indices order -- a uint8 torch tensor of
    m*24 bytes (device-resident from api.price_american_tc_batch) or a numpy
    QUOTE_DTYPE array.  Returns the whole batch's quotes (numpy QUOTE_DTYPE) on
    every rank."""
    import torch
    import torch.distributed as dist
    counts = np.bincount(rank_of, minlength=nranks)
    M = int(counts.max()) if len(counts) else 0
    if device is None:
        device = local.device if isinstance(local, torch.Tensor) else torch.device("cpu")
    if not isinstance(local, torch.Tensor):
        local = torch.from_numpy(np.ascontiguousarray(local).view(np.uint8).copy())
    m = int(counts[rank])
    assert local.numel() == m * QUOTE_BYTES, (local.numel(), m)
    buf = torch.zeros(max(M, 1) * QUOTE_BYTES, dtype=torch.uint8, device=device)
    buf[: m * QUOTE_BYTES] = local.to(device)
    allb = torch.empty(nranks * buf.numel(), dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(allb, buf, group=group)
    host = allb.cpu().numpy()
    out = np.empty(len(rank_of), dtype=api.QUOTE_DTYPE)
    stride = max(M, 1) * QUOTE_BYTES
    for g in range(nranks):
        idx = local_indices(rank_of, g)
        seg = host[g * stride: g * stride + len(idx) * QUOTE_BYTES]
        out[idx] = seg.view(api.QUOTE_DTYPE)
    return out


def price_batch_sharded(batch, N: int, rank: int, nranks: int, group=None, pricer=None):
    """Price one batch over `nranks` ranks; every rank calls it with the same
    batch.  pricer(sub_batch, N) -> QUOTE_DTYPE array or uint8 device tensor
    (default: the CUDA batch API on this rank's current device).  Returns
    (quotes of the whole batch in batch order, this rank's index set)."""
    rank_of, _ = plan(batch, N, nranks)
    idx = local_indices(rank_of, rank)
    sub = batch.subset(idx)
    if pricer is None:
        out, _rc = api.price_american_tc_batch(api.device_batch(sub), N)
        local = out
    else:
        local = pricer(sub, N)
    return gather_quotes(local, rank_of, rank, nranks, group=group), idx
