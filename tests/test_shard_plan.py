"""CPU (gloo, world size 2 and 3) check of the single-tree sharding scheme of
amtc_price_tree_sharded (paper_1110_2477_b200/csrc/amtc_tree.cu): columns
[ceil(g w/n_act), ceil((g+1) w/n_act)) on the first n_act = clamp(w / mc, 1, n)
ranks (processor reduction), re-split every band of D levels, window
= own new range + D halo columns, gathered by point-to-point transfers from the
owners.  The band recurrence here is a numpy stand-in (test infrastructure);
the result must equal the oracle's CRR price, and every window column must be
received exactly once."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


MIN_COLS = 4096  # amtc_tree.cu TREE_MIN_COLS (processor reduction)


def split_at(w, g, n, min_cols=MIN_COLS):
    na = max(1, min(n, w // min_cols))
    if g >= na:
        return w
    return (g * w + na - 1) // na


def need(w0, w1, Dp, g, n, mc=MIN_COLS):
    a0, b0 = split_at(w0, g, n, mc), split_at(w0, g + 1, n, mc)
    return a0, (min(b0 + Dp, w1) if b0 > a0 else a0)


def _worker(rank, world, port, N, D, mc, opt, out_q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    u = np.exp(opt.sigma * np.sqrt(opt.T / N)); d = 1 / u; r = np.exp(opt.R * opt.T / N)
    p = (r - d) / (u - d); pu, pd = p / r, (1 - p) / r
    ex = lambda t, j: np.maximum(opt.K - opt.S0 * u ** (t - 2 * j), 0.0)  # put
    a, b = split_at(N + 1, rank, world, mc), split_at(N + 1, rank + 1, world, mc)
    cur = ex(N, np.arange(a, b, dtype=np.float64))
    t_top = N
    while t_top > 0:
        Dp = min(D, t_top); t_bot = t_top - Dp
        w1, w0 = t_top + 1, t_bot + 1
        lo, hi = need(w0, w1, Dp, rank, world, mc)
        win = np.full(hi - lo, np.nan)
        got = np.zeros(hi - lo, dtype=np.int64)
        reqs = []
        for h in range(world):
            ha, hb = split_at(w1, h, world, mc), split_at(w1, h + 1, world, mc)
            if h == rank:
                for g in range(world):
                    if g == rank:
                        continue
                    glo, ghi = need(w0, w1, Dp, g, world, mc)
                    x0, x1 = max(glo, ha), min(ghi, hb)
                    if x1 > x0:
                        reqs.append(dist.isend(torch.from_numpy(cur[x0 - ha:x1 - ha].copy()), g))
            else:
                x0, x1 = max(lo, ha), min(hi, hb)
                if x1 > x0:
                    buf = torch.empty(x1 - x0, dtype=torch.float64)
                    dist.recv(buf, h)
                    win[x0 - lo:x1 - lo] = buf.numpy(); got[x0 - lo:x1 - lo] += 1
        x0, x1 = max(lo, a), min(hi, b)
        if x1 > x0:
            win[x0 - lo:x1 - lo] = cur[x0 - a:x1 - a]; got[x0 - lo:x1 - lo] += 1
        for q in reqs:
            q.wait()
        assert np.all(got == 1), (rank, t_top, got)
        # band: Dp levels on the window, keep the new own range
        v = win.copy()
        for t in range(t_top - 1, t_bot - 1, -1):
            j = lo + np.arange(len(v) - 1)
            v = np.maximum(ex(t, j), pu * v[:-1] + pd * v[1:])
        a0, b0 = split_at(w0, rank, world, mc), split_at(w0, rank + 1, world, mc)
        cur = v[: b0 - a0]
        a, b = a0, b0
        t_top = t_bot
    if rank == 0:
        out_q.put(float(cur[0]))
    dist.barrier()
    dist.destroy_process_group()


# mc: the processor-reduction threshold (columns per active rank; 4096 in the
# library) scaled down so that small trees exercise both the distribution and
# the reduction to fewer ranks near the root
@pytest.mark.parametrize("world,N,D,mc", [(2, 300, 16, 40), (3, 257, 32, 24), (2, 40, 128, 8), (3, 200, 16, 1)])
def test_sharded_scheme_gloo(world, N, D, mc):
    opt = O.Option(100.0, 100.0, 1.0, 0.3, 0.05, 0.0, O.PUT)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + world * 7 + N % 13
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, D, mc, opt, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    price = q.get(timeout=10)
    ref = O.price_crr(opt, N)
    assert abs(price - ref) <= 1e-9 * abs(ref)
