"""CPU (gloo, world size 2 and 3) run of the single-tree sharding of
amtc_price_tree_sharded (paper_1110_2477_b200/csrc/amtc_tree.cu) driven by the
LIBRARY's own exchange plan (amtc_tree_band_plan, the function tree_run calls
before every band): columns [ceil(g w/n_act), ceil((g+1) w/n_act)) on the first
n_act = clamp(w / mc, 1, n) ranks (processor reduction), re-split
every band of D levels, window = own new range + D halo columns
(region-B dependency), gathered by point-to-point transfers.  Only
the band recurrence is a numpy stand-in (test infrastructure) for the GPU band
kernel; the result must equal the oracle's CRR price and every window column
must be received exactly once."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _worker(rank, world, port, N, D, mc, opt, out_q):
    import torch
    from paper_1110_2477_b200 import api
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    u = np.exp(opt.sigma * np.sqrt(opt.T / N)); d = 1 / u; r = np.exp(opt.R * opt.T / N)
    p = (r - d) / (u - d); pu, pd = p / r, (1 - p) / r
    ex = lambda t, j: np.maximum(opt.K - opt.S0 * u ** (t - 2 * j), 0.0)  # put
    nb = api.tree_band_plan(N, world, rank, -1, D, mc)
    cur = None
    for band in range(nb):
        P, snd, rcv = api.tree_band_plan(N, world, rank, band, D, mc)
        t_top, Dp = P["t_top"], P["Dp"]
        a, b, lo, hi = P["own_lo"], P["own_hi"], P["win_lo"], P["win_hi"]
        if band == 0:
            cur = ex(N, np.arange(a, b, dtype=np.float64))
        assert len(cur) == b - a
        assert max(b - a, hi - lo, P["new_hi"] - P["new_lo"]) <= P["cap"]
        win = np.full(hi - lo, np.nan)
        got = np.zeros(hi - lo, dtype=np.int64)
        reqs = []
        for g in range(world):
            if g == rank:
                continue
            s0, s1 = snd[g]
            if s1 > s0:
                reqs.append(dist.isend(torch.from_numpy(cur[s0 - a:s1 - a].copy()), g))
        for g in range(world):
            if g == rank:
                continue
            r0, r1 = rcv[g]
            if r1 > r0:
                buf = torch.empty(r1 - r0, dtype=torch.float64)
                dist.recv(buf, g)
                win[r0 - lo:r1 - lo] = buf.numpy(); got[r0 - lo:r1 - lo] += 1
        x0, x1 = max(lo, a), min(hi, b)
        if x1 > x0:
            win[x0 - lo:x1 - lo] = cur[x0 - a:x1 - a]; got[x0 - lo:x1 - lo] += 1
        for q in reqs:
            q.wait()
        assert np.all(got == 1), (rank, t_top, got)
        # band: Dp levels on the window, keep the new own range
        v = win.copy()
        for t in range(t_top - 1, t_top - Dp - 1, -1):
            j = lo + np.arange(len(v) - 1)
            v = np.maximum(ex(t, j), pu * v[:-1] + pd * v[1:])
        cur = v[: P["new_hi"] - P["new_lo"]]
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


@pytest.mark.parametrize("N,world", [(5000, 2), (8191, 8), (12000, 3), (100000, 8), (100000, 2), (300, 8),
                                     (1000000, 8)])
def test_band_plan_fits_buffers_and_partitions(N, world):
    """With the library's own band depth and threshold: for every band and rank
    the own range, the new range and the window fit the level buffers (`cap`;
    ADVICE r1: N = 5000 on 2 ranks keeps 5001 columns on rank 0), the ranks'
    ranges partition each level, every send matches the peer's receive, and the
    windows cover exactly the dependency cone [new_lo, min(new_hi + Dp, w))."""
    from paper_1110_2477_b200 import api
    nb = api.tree_band_plan(N, world, 0)
    assert nb == (N + 255) // 256
    for band in range(0, nb, max(1, nb // 50)):
        plans = [api.tree_band_plan(N, world, g, band) for g in range(world)]
        t_top, Dp = plans[0][0]["t_top"], plans[0][0]["Dp"]
        w1, w0 = t_top + 1, t_top - Dp + 1
        own = sorted((P["own_lo"], P["own_hi"]) for P, _, _ in plans)
        new = sorted((P["new_lo"], P["new_hi"]) for P, _, _ in plans)
        assert own[0][0] == 0 and own[-1][1] == w1 and all(own[i][1] == own[i + 1][0] for i in range(world - 1))
        assert new[0][0] == 0 and new[-1][1] == w0 and all(new[i][1] == new[i + 1][0] for i in range(world - 1))
        for g, (P, snd, rcv) in enumerate(plans):
            assert max(P["own_hi"] - P["own_lo"], P["win_hi"] - P["win_lo"], P["new_hi"] - P["new_lo"]) <= P["cap"]
            if P["new_hi"] > P["new_lo"]:
                assert (P["win_lo"], P["win_hi"]) == (P["new_lo"], min(P["new_hi"] + Dp, w1))
            for h in range(world):
                if h != g:
                    assert tuple(snd[h]) == tuple(plans[h][2][g])  # g's send to h == h's receive from g
