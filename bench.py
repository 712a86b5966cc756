#!/usr/bin/env python
"""Benchmark of the amtc hot path (BASELINE.json metric) -- one JSON line.

Default workload (BASELINE.json config 4): 16384 American options per GPU
(45% put, 45% call, 10% bull spread; seeded synthetic), N = 1500 steps, ask AND
bid under proportional costs k ~ U[0, 2%], fp64.  One "step" = pricing the
whole batch through the C-ABI (amtc_price_american_tc_batch, inputs resident in
HBM).  Multi-GPU: one process per GPU (torchrun); each rank prices its own
ONE 16384-option batch is dealt over the ranks by amtc_batch_shard_plan
(cost-sorted snake order, equal counts) and the 24-byte quotes are all-gathered
at the end of every step -> strong scaling; timing = max over ranks of the
device time (CUDA events), value = the batch's node-updates / that time.
--slice g/n times rank g's share of an n-GPU deal alone on one GPU (per-rank
times of an n-GPU run without n GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4|2] [--impl amtc|reference]

--impl reference times the CPU oracle (oracle/, plain C) on a bounded sample of
the same workload on this host's cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]

# FP64 roofline: 148 SMs x 64 FP64 lanes/clk x 2 flop/FMA x clock (B200_PROFILING.md
# unit counts; MEASURED_PEAKS.json has no FP64 figure).  See DESIGN.md "Roofline".
FP64_LANES_PER_SM = 64
# algorithmic FP64 cost model: 12 flop per child vertex per node-update
TC_FLOP_PER_CHILD_VERTEX = 12.0
CRR_FLOP_PER_NODE = 6.0  # DFMA(X) + DMUL + DFMA + DMNMX = 2 + 1 + 2 + 1


def tc_nodes(N: int) -> int:
    """node-updates per option at levels 0..N: (N+1)(N+2)/2."""
    return (N + 1) * (N + 2) // 2


def crr_nodes(N: int) -> int:
    return N * (N + 1) // 2


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def flush_l2(buf):
    buf.add_(1.0)  # 512 MiB read+write > 126 MB L2


def setup_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if __import__("torch").cuda.is_available() else "gloo")
        pg = dist
    return world, rank, local, pg


def max_over_ranks(x: float, pg, device) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, pg, device) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def workload(config: int, rank: int = 0):
    """ONE seeded batch of the workload; under torchrun every rank draws the same
    batch and prices the share amtc_batch_shard_plan deals it (strong scaling)."""
    from paper_1110_2477_b200 import workloads as W
    if config == 4:
        return W.config4(), W.CONFIG4_N, "config4: American put/call/bull-spread batch, ask+bid under proportional costs"
    if config == 2:
        return W.config2(), W.CONFIG2_N, "config2: zero-cost American put/call batch (CRR), one tree per warp"
    raise SystemExit(f"unknown --config {config}")


def oracle_cache(config: int, batch):
    """The cached full-batch oracle file (tests/golden/oracle_config<c>_full.npz,
    written by scripts/make_full_refs.py from oracle/ only), if its SHA-256 key
    matches this batch; else None."""
    from paper_1110_2477_b200 import workloads as W
    path = os.path.join(ROOT, "tests", "golden", f"oracle_config{config}_full.npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    if str(z["sha256"]) != W.soa_sha256(batch):
        return None
    return z


# A19: |g - o| <= 1e-9 |o|, or the rounding floor 4 N eps S0
REL_TOL = 1e-9
FLOOR_C = 4.0


def abs_floor(N: int, S0) -> np.ndarray:
    """DESIGN.md A19: FLOOR_C N eps S0 (N levels of fp64 updates of values of size S0)."""
    return FLOOR_C * N * np.finfo(np.float64).eps * np.asarray(S0, dtype=np.float64)


def parity_vs_oracle(got: np.ndarray, ref: np.ndarray, N: int, S0) -> dict:
    """Element-wise comparison with the cached oracle (every option)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    rel_ok = err <= REL_TOL * np.abs(ref)
    floor_ok = err <= abs_floor(N, np.broadcast_to(S0, ref.shape))
    ok = rel_ok | floor_ok
    nz = np.abs(ref) > 0
    return {"checked": int(ref.size), "pass": int(ok.sum()), "fail": int((~ok).sum()),
            "max_rel_err": float(np.max(err[nz] / np.abs(ref[nz]))) if nz.any() else 0.0,
            "max_err_over_N_eps_S0": float(np.max(err / abs_floor(N, np.broadcast_to(S0, ref.shape)) * FLOOR_C)),
            "floor_used": int((floor_ok & ~rel_ok).sum())}


def cpu_baseline(config: int, budget_options: int = 24, seed: int = 123) -> dict:
    """The oracle as it stands, on all host cores, on a bounded seeded sample.
    With the cached oracle op counts available the sample's throughput is
    extrapolated by WORK (the SURVEY 8(d) cost-model ops of the sample vs the
    whole batch), so the value does not hinge on how many heavy call buyers the
    sample happens to hold."""
    import oracle as O
    b, N, _ = workload(config, 0)
    g = np.random.default_rng(seed)
    idx = np.sort(g.choice(len(b), budget_options, replace=False))
    cores = len(os.sched_getaffinity(0))
    opts = []
    for i in idx:
        r = b.row(int(i))
        opts.append(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], r["k"], r["kind"], r["K2"]))
    t0 = time.perf_counter()
    if config == 4:
        O.price_tc_many(opts, N, threads=cores)
        nodes = tc_nodes(N) * len(opts)
    else:
        O.price_crr_many(opts, N, threads=cores)
        nodes = crr_nodes(N) * len(opts)
    dt = time.perf_counter() - t0
    raw = nodes / dt
    value, how = raw, "per option"
    z = oracle_cache(config, b) if config == 4 else None
    if z is not None:
        ops = z["fp64_ops"].astype(np.float64)
        # time for the whole batch at the sample's ops/s; value = batch node-updates / that
        t_batch = dt * ops.sum() / ops[idx].sum()
        value, how = tc_nodes(N) * len(b) / t_batch, "by oracle cost-model ops (sample ops / batch ops)"
    return {"value": value, "unit": "node-updates/s", "cores": min(cores, len(opts)), "kind": "oracle",
            "sample": f"{len(opts)} options of the config-{config} batch (numpy default_rng({seed}) choice), "
                      f"N={N}, one option per thread on {min(cores, len(opts))} threads, {dt:.1f} s wall; "
                      f"extrapolated {how}",
            "raw_sample_value": raw, "options_per_s": value / (tc_nodes(N) if config == 4 else crr_nodes(N))}


def run_reference(args):
    world, rank, local, pg = setup_dist()
    if rank != 0:
        return 0
    times = []
    for i in range(args.warmup + args.steps):
        res = cpu_baseline(args.config, budget_options=args.ref_options, seed=123 + i)
        if i >= args.warmup:
            times.append(res)
    vals = [r["value"] for r in times]
    value = float(np.mean(vals))
    b, N, desc = workload(args.config, 0)
    per_opt = tc_nodes(N) if args.config == 4 else crr_nodes(N)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "node-updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(len(b) * per_opt / value * 1e3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "N": N, "options_total": len(b),
                       "node_updates_per_option": per_opt,
                       "parallelism": "host cores, one option per thread",
                       "reference_sample": f"each step prices a seeded sample of {args.ref_options} options of "
                                           "this workload (bounded CPU time); ms_per_step is the whole batch "
                                           "at that rate"},
            "cpu_baseline": {"value": value, "unit": "node-updates/s", "cores": times[-1]["cores"],
                             "kind": "oracle", "sample": times[-1]["sample"]},
            "e2e": {"value": value, "unit": "node-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def fp64_peak():
    """FP64 DFMA peak measured on this pool (tools/fp64_peak.cu ->
    profiles/r01_fp64_peak.json): instr/s and flop/s; else the unit-count value."""
    f = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    try:
        m = json.load(open(f))
        tf = float(m["fp64_tflops"])
        return tf * 1e12 / 2.0, tf * 1e12, ("measured: DFMA throughput by tools/fp64_peak.cu on this pool's "
                                            "B200 (profiles/r01_fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry)")
    except Exception:
        v = 148 * FP64_LANES_PER_SM * 1965e6
        return v, 2 * v, "derived: 148 SMs x 64 FP64 lanes/clk x 1965 MHz (no measurement found)"


def max_bp_hist(mbp: np.ndarray) -> dict:
    edges = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]
    out = {}
    lo = 0
    for e in edges:
        c = int(((mbp >= lo) & (mbp < e)).sum()) if lo else int((mbp < e).sum())
        out[f"<{e}"] = c
        lo = e
    out[f">={edges[-1]}"] = int((mbp >= edges[-1]).sum())
    return out


def run_amtc(args):
    import torch
    world, rank, local, pg = setup_dist()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1110_2477_b200 import api, build
    build.build()
    api.lib()
    b, N, desc = workload(args.config)
    # the deal: this rank's share of ONE batch (--slice g/n: rank g's share of an
    # n-GPU deal, timed alone on this one GPU)
    g_eff, n_eff = rank, world
    if args.slice:
        assert world == 1, "--slice runs one share on one GPU"
        g_eff, n_eff = (int(x) for x in args.slice.split("/"))
    rank_of, est_cost = api.batch_shard_plan(b, N, n_eff)
    idx = np.nonzero(rank_of == g_eff)[0]
    sub = b.subset(idx)
    n = len(sub)
    cols = api.device_batch(sub, dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    counts = np.bincount(rank_of, minlength=n_eff)
    M = int(counts.max())
    qbytes = 24 if args.config == 4 else 8
    if args.config == 4:
        out = torch.empty(n * 24, dtype=torch.uint8, device=dev)
        price = lambda: api.price_american_tc_batch(cols, N, out, stream)
        per_opt = tc_nodes(N)
    else:
        out = torch.empty(n * 8, dtype=torch.uint8, device=dev)
        out64 = out.view(torch.float64)
        price = lambda: api.price_crr_batch(cols, N, out64, stream)
        per_opt = crr_nodes(N)
    nodes_per_step = per_opt * len(b) if not args.slice else per_opt * n
    gbuf = torch.zeros(M * qbytes, dtype=torch.uint8, device=dev)
    gall = torch.empty(world * M * qbytes, dtype=torch.uint8, device=dev)

    def step():
        price()
        if pg is not None:  # the final gather of the quotes (the only inter-GPU traffic)
            gbuf[: n * qbytes].copy_(out)
            pg.all_gather_into_tensor(gall, gbuf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = api.launch_count()
    full_ms, light_ms = 0.0, 0.0
    for i in range(args.steps):
        flush_l2(flush)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
        if args.config == 4:
            st = api.tc_last_stats()
            full_ms += st["full_ms"]
            light_ms += st["light_ms"]
    torch.cuda.synchronize()
    launches = api.launch_count() - launches0
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    my_ms = float(np.sum(step_ms))
    rank_ms = [my_ms]
    if pg is not None:
        t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
        tl = [torch.empty_like(t) for _ in range(world)]
        pg.all_gather(tl, t)
        rank_ms = [float(x.item()) for x in tl]
    total_ms = max(rank_ms)
    value = nodes_per_step * args.steps / (total_ms / 1e3)

    # the gathered quotes, in batch order, for parity and the max_bp histogram
    if pg is not None:
        host = gall.cpu().numpy()
        res = np.empty(len(b), dtype=api.QUOTE_DTYPE if args.config == 4 else np.float64)
        for g in range(world):
            ig = np.nonzero(rank_of == g)[0]
            seg = host[g * M * qbytes: g * M * qbytes + len(ig) * qbytes]
            res[ig] = seg.view(res.dtype)
        res_idx = np.arange(len(b))
    else:
        res = out.cpu().numpy().view(api.QUOTE_DTYPE if args.config == 4 else np.float64)
        res_idx = idx

    # parity of this step's output against the cached oracle (every option priced)
    parity = None
    z = oracle_cache(args.config, b)
    if z is not None and rank == 0:
        if args.config == 4:
            pa = parity_vs_oracle(res["ask"], z["ask"][res_idx], N, b.S0[res_idx])
            pb = parity_vs_oracle(res["bid"], z["bid"][res_idx], N, b.S0[res_idx])
            parity = {"ask": pa, "bid": pb, "source": "tests/golden/oracle_config4_full.npz (oracle/, SHA-256 keyed)",
                      "tolerance": "A19: 1e-9 relative, or the rounding floor 4 N eps S0 (counted)"}
        else:
            parity = {"price": parity_vs_oracle(res, z["price"][res_idx], N, b.S0[res_idx]),
                      "source": "tests/golden/oracle_config2_full.npz (oracle/, SHA-256 keyed)",
                      "tolerance": "A19: 1e-9 relative, or the rounding floor 4 N eps S0 (counted)"}

    # roofline: algorithmic FP64 work from the ORACLE's cost-model counts (cached per option)
    instr_peak, flop_peak, peak_src = fp64_peak()
    roofline = None
    if args.config == 4:
        if z is not None:
            # the prepare kernel's item classes (amtc_prepare.cu item_class): the light
            # kernel takes put sellers, call sellers with k/h < 4 and put buyers
            kh = b.k[idx] / (b.sigma[idx] * np.sqrt(b.T[idx] / N))
            seller_light = (b.kind[idx] == 0) | ((b.kind[idx] == 1) & (kh < 4.0))
            buyer_light = b.kind[idx] == 0
            ops_a = z["fp64_ops_ask"][idx].astype(np.float64)
            ops_b = z["fp64_ops_bid"][idx].astype(np.float64)
            light_ops = ops_a[seller_light].sum() + ops_b[buyer_light].sum()
            full_ops = ops_a[~seller_light].sum() + ops_b[~buyer_light].sum()
            fm, lm = full_ms / args.steps, light_ms / args.steps
            per_k = {}
            for name, ops, ms in (("full", full_ops, fm), ("light", light_ops, lm)):
                if ms > 0:
                    a = ops / (ms / 1e3)
                    per_k[name] = {"ops_per_step": ops, "ms": ms, "achieved_instr_per_s": a,
                                   "frac_of_dfma_instr_peak": a / instr_peak, "frac_of_flop_peak": a / flop_peak}
            ach = full_ops / (fm / 1e3) if fm > 0 else 0.0
            roofline = {"bound": "alu", "achieved": ach / 1e12, "peak": instr_peak / 1e12,
                        "unit": "T FP64-instr/s", "frac": ach / instr_peak,
                        "traffic": None, "kernel": "strip_kernel<3,3,20,1,1> (full; the dominant kernel)",
                        "kernels": per_k,
                        "work_source": "oracle cost-model ops (SURVEY 8(d): merge 3, crossing 4, restriction 2|4, "
                                       "scaling 2) per option and party, tests/golden/oracle_config4_full.npz",
                        "peak_source": peak_src + "; DFMA = 1 instruction (the cost model counts instructions)",
                        "flop_peak_tflops": flop_peak / 1e12}
            # the committed ncu launch list of this command (serialised, cold cache): each
            # kernel's share of the step, to compare with the live event times above
            lf = os.path.join(ROOT, "profiles", "r02_launches_config4.csv")
            if os.path.exists(lf):
                try:
                    import csv as _csv
                    rows = [r for r in _csv.reader(open(lf)) if len(r) > 10]
                    ki, vi = rows[0].index("Kernel Name"), rows[0].index("Metric Value")
                    tot, per = 0.0, {}
                    for r in rows[1:]:
                        ns = float(r[vi].replace(",", ""))
                        tot += ns
                        key = "full" if "strip_kernel" in r[ki] or "full_kernel" in r[ki] else (
                            "light" if "light_kernel" in r[ki] else "other")
                        per[key] = per.get(key, 0.0) + ns
                    roofline["launch_list"] = {k: {"share": v / tot, "ns_total": v} for k, v in per.items()}
                    roofline["launch_list_source"] = "profiles/r02_launches_config4.csv (ncu gpu__time_duration.sum, serialised)"
                except Exception:
                    pass
            if "light" in per_k:
                per_k["light"]["note"] = ("event span on the second stream: includes the wait for SMs the full kernel "
                                          "holds (its CTAs take ~210 KB of shared memory), so it overstates the light "
                                          "kernel's run time; the launch list's serialised time is the kernel's own")
            tf = os.path.join(ROOT, "profiles", "r02_traffic_config4.json")
            if os.path.exists(tf):
                try:
                    tj = json.load(open(tf))
                    roofline["traffic"] = float(tj["full_kernel_bytes"])
                    roofline["traffic_source"] = tj.get("source", tf)
                except Exception:
                    pass
    else:
        kern_ms = float(np.mean(step_ms))
        ops = 3.0 * per_opt * n   # 1 DMUL + 1 DFMA + 1 DMNMX per CRR node-update
        a = ops / (kern_ms / 1e3)
        roofline = {"bound": "alu", "achieved": a / 1e12, "peak": instr_peak / 1e12, "unit": "T FP64-instr/s",
                    "frac": a / instr_peak, "traffic": None, "kernel": "crr_kernel",
                    "work_source": "SURVEY 8(d): 3 FP64-pipe instructions per CRR node-update",
                    "peak_source": peak_src}

    # end to end through the public C-ABI with HOST buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        pinned = {f: torch.from_numpy(np.ascontiguousarray(getattr(sub, f))).pin_memory()
                  for f in ("S0", "K", "K2", "T", "sigma", "R", "k", "kind")}
        hb = {f: t.numpy() for f, t in pinned.items()}
        h2d = sum(t.numel() * t.element_size() for t in pinned.values())
        e2e_steps = max(1, min(args.steps, 3))
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            if args.config == 4:
                q, rc = api.price_american_tc_batch_host(hb, N, stream)
            else:
                q = api.price_crr_batch_host(hb, N, stream)
            d2h = q.nbytes
            if pg is not None:
                gbuf[: n * qbytes].copy_(torch.from_numpy(q.view(np.uint8)).to(dev))
                pg.all_gather_into_tensor(gall, gbuf)
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, pg, dev)
        e2e = {"value": nodes_per_step * e2e_steps / e2e_s,
               "unit": "node-updates/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e2e_steps, "timer": "host wall clock around the synchronous C-ABI call (+ the quote gather)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.slice:
        cpu = cpu_baseline(args.config, budget_options=args.ref_options)

    if rank == 0:
        par = (f"dp{world}: one batch dealt by amtc_batch_shard_plan (cost-sorted snake order), "
               "no inter-GPU traffic but a final all-gather of the quotes")
        line = {"metric": METRIC, "value": value, "unit": "node-updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": desc, "N": N, "options_total": len(b),
                           "options_per_rank": [int(c) for c in counts],
                           "options_per_s": (len(b) if not args.slice else n) * args.steps / (total_ms / 1e3),
                           "node_updates_per_option": per_opt,
                           "l2": "flushed before every timed step (512 MiB write, untimed)",
                           "parallelism": par},
                "rank_ms_per_step": [r_ / args.steps for r_ in rank_ms],
                "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks, "step_ms": step_ms}
        if args.config == 4:
            line["max_bp_hist"] = max_bp_hist(np.asarray(res["max_bp"]))
        if args.slice:
            line["slice"] = {"rank": g_eff, "of": n_eff, "options": n,
                             "est_cost_share": float(est_cost[g_eff] / est_cost.sum()),
                             "note": "one rank's share of the n-GPU deal, timed alone on one GPU"}
            line["config"]["workload"] = desc + f" -- slice {g_eff}/{n_eff} of the deal"
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def run_tree(args):
    """Configs 1, 3, 5 (single trees).  Config 5a (CRR, N = 100000) runs sharded
    over all ranks through amtc_price_tree_sharded (NCCL halo exchange, strong
    scaling); configs 1, 3 and 5b run the north-star single-option call (strip-
    split mode) on rank 0.  Timer: host wall clock around the synchronous C-ABI
    calls (they include the host-side band loop), max over ranks."""
    import torch
    from paper_1110_2477_b200 import api, build, workloads as W
    world, rank, local, pg = setup_dist()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    build.build()
    api.lib()
    comm = None
    if args.config == 5:
        r = W.config5a().row(0)
        N = W.CONFIG5A_N
        if world > 1:
            comm, _, _ = api.comm_from_torch_dist()
        def step():
            q = api.price_tree_sharded(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, 0.0, api.PUT,
                                       comm=comm, rank=rank, nranks=world)
            assert q["status"] == 0, q
        nodes = crr_nodes(N)
        desc = f"config5a: one American put tree, k=0 CRR, N={N}, sharded over {world} GPU(s) (NCCL halo per band)"
        scaling = "strong"
        cpu_sample = (dict(S0=r["S0"], K=r["K"], T=r["T"], sigma=r["sigma"], R=r["R"], k=0.0, kind=0), 20000, "crr")
    else:
        if args.config == 1:
            trees = [(W.config1().row(0), W.CONFIG1_N)]
            desc = "config1: Example 5.1 put, N=100, ask+bid (north-star single call)"
        else:
            trees = [(b.row(0), N_) for b, N_ in W.config3()]
            desc = ("config3: put+call x k in {0,.0025,.005,.01,.02} x N in {250..2000}, 50 single trees, "
                    "one batched call per N (10 trees, strip-split mode: intra-tree parallel)")
        groups = {}
        for b, N_ in ([(W.config1(), W.CONFIG1_N)] if args.config == 1 else W.config3()):
            groups.setdefault(N_, []).append(b)
        batches = {N_: W.concat(bs) for N_, bs in groups.items()}
        def step():
            if rank != 0:
                return
            if args.config == 1:
                row, N_ = trees[0]
                q = api.price_american_tc(row["S0"], row["K"], row["T"], row["sigma"], row["R"], N_, row["k"],
                                          row["kind"], row["K2"])
                assert q["status"] == 0, q
                return
            for N_, bb in batches.items():
                q, rc = api.price_american_tc_batch_host(bb, N_)
                assert rc == 0, rc
        nodes = sum(tc_nodes(N_) for _, N_ in trees)
        scaling = "weak"
        row0, N0 = trees[0]
        cpu_sample = (dict(S0=row0["S0"], K=row0["K"], T=row0["T"], sigma=row0["sigma"], R=row0["R"], k=row0["k"],
                           kind=row0["kind"], K2=row0["K2"]), N0, "tc")
        N = max(N_ for _, N_ in trees)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
    times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    clocks = sampler.stop() if sampler else None
    tot = max_over_ranks(float(np.sum(times)), pg, dev)
    value = nodes * args.steps / tot
    extra = None
    if args.config == 5:
        # config 5b: the transaction-cost tree, sharded the same way (k > 0 path)
        r5 = W.config5b().row(0)
        def step5b():
            q = api.price_tree_sharded(r5["S0"], r5["K"], r5["T"], r5["sigma"], r5["R"], W.CONFIG5B_N, r5["k"],
                                       api.PUT, comm=comm, rank=rank, nranks=world)
            assert q["status"] == 0, q
            return q
        step5b()
        torch.cuda.synchronize()
        t5 = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            q5 = step5b()
            torch.cuda.synchronize()
            t5.append(time.perf_counter() - t0)
        tot5 = max_over_ranks(float(np.sum(t5)), pg, dev)
        extra = {"config5b": {"N": W.CONFIG5B_N, "k": r5["k"], "ms_per_step": 1e3 * tot5 / args.steps,
                              "node_updates_per_s": tc_nodes(W.CONFIG5B_N) * args.steps / tot5,
                              "ask": q5["ask"], "bid": q5["bid"]}}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle as O_  # the cpu_baseline leg only
        params, Ns, kind = cpu_sample
        opt = O_.Option(**params)
        t0 = time.perf_counter()
        if kind == "crr":
            O_.price_crr(opt, Ns)
            cn = crr_nodes(Ns)
        else:
            O_.price_tc(opt, Ns)
            cn = tc_nodes(Ns)
        dt = time.perf_counter() - t0
        cpu = {"value": cn / dt, "unit": "node-updates/s", "cores": 1, "kind": "oracle",
               "sample": f"one tree of the workload at N={Ns}, single thread, {dt:.2f} s"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "node-updates/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "N": N, "node_updates_per_step": nodes,
                           "timer": "host wall clock around synchronous C-ABI calls, max over ranks",
                           "l2": "inputs are scalars; levels live in HBM/L2 between bands"},
                "roofline": None, "cpu_baseline": cpu, "e2e": None, "clocks": clocks,
                "step_ms": [1e3 * t for t in times]}
        if extra:
            line["extra"] = extra
        print(json.dumps(line), flush=True)
    if comm is not None:
        api.comm_destroy(comm)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="amtc", choices=["amtc", "reference"])
    ap.add_argument("--ref-options", type=int, default=24)
    ap.add_argument("--slice", default=None, help="g/n: time rank g's share of an n-GPU deal on this GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config in (1, 3, 5):
        return run_tree(args)
    return run_amtc(args)


if __name__ == "__main__":
    sys.exit(main())
