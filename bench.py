#!/usr/bin/env python
"""Benchmark of the amtc hot path (BASELINE.json metric) -- one JSON line.

Default workload (BASELINE.json config 4): 16384 American options per GPU
(45% put, 45% call, 10% bull spread; seeded synthetic), N = 1500 steps, ask AND
bid under proportional costs k ~ U[0, 2%], fp64.  One "step" = pricing the
whole batch through the C-ABI (amtc_price_american_tc_batch, inputs resident in
HBM).  Multi-GPU: one process per GPU (torchrun); each rank prices its own
16384-option batch (seed + rank) with no data-path collective -> weak scaling;
timing = max over ranks of the device time (CUDA events), whole-job value =
all ranks' node-updates / that time.

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


def workload(config: int, rank: int):
    from paper_1110_2477_b200 import workloads as W
    if config == 4:
        b = W.config4(seed=W.SEED_BASE + 4 + 1000 * rank)
        return b, W.CONFIG4_N, "config4: American put/call/bull-spread batch, ask+bid under proportional costs"
    if config == 2:
        b = W.config2(seed=W.SEED_BASE + 2 + 1000 * rank)
        return b, W.CONFIG2_N, "config2: zero-cost American put/call batch (CRR), one tree per warp"
    raise SystemExit(f"unknown --config {config}")


def cpu_baseline(config: int, budget_options: int = 8, seed: int = 123) -> dict:
    """The oracle as it stands, on all host cores, on a bounded seeded sample."""
    import oracle as O
    from paper_1110_2477_b200 import workloads as W
    b, N, _ = workload(config, 0)
    idx = np.sort(np.random.default_rng(seed).choice(len(b), budget_options, replace=False))
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
    return {"value": nodes / dt, "unit": "node-updates/s", "cores": min(cores, len(opts)), "kind": "oracle",
            "sample": f"{len(opts)} options of the config-{config} batch (numpy default_rng({seed}) choice), "
                      f"N={N}, one option per thread, {dt:.1f} s wall",
            "options_per_s": len(opts) / dt}


def run_reference(args):
    world, rank, local, pg = setup_dist()
    if rank != 0:
        return 0
    times = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_baseline(args.config, budget_options=args.ref_options, seed=123 + i)
        if i >= args.warmup:
            times.append(res)
    vals = [r["value"] for r in times]
    value = float(np.mean(vals))
    b, N, desc = workload(args.config, 0)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "node-updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean([args.ref_options * tc_nodes(N) / r["value"] * 1e3 for r in times])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "N": N, "options_per_gpu": len(b), "options_total": len(b),
                       "node_updates_per_option": tc_nodes(N) if args.config == 4 else crr_nodes(N),
                       "parallelism": "host cores, one option per thread",
                       "reference_sample": f"each step prices a seeded sample of {args.ref_options} options of "
                                           "this workload (bounded CPU time)"},
            "cpu_baseline": {"value": value, "unit": "node-updates/s", "cores": times[-1]["cores"],
                             "kind": "oracle", "sample": times[-1]["sample"]},
            "e2e": {"value": value, "unit": "node-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_amtc(args):
    import torch
    world, rank, local, pg = setup_dist()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1110_2477_b200 import api, build
    build.build()
    api.lib()
    b, N, desc = workload(args.config, rank)
    n = len(b)
    cols = api.device_batch(b, dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    if args.config == 4:
        out = torch.empty(n * 24, dtype=torch.uint8, device=dev)
        step = lambda: api.price_american_tc_batch(cols, N, out, stream)
        nodes_per_step = tc_nodes(N) * n
    else:
        out = torch.empty(n, dtype=torch.float64, device=dev)
        step = lambda: api.price_crr_batch(cols, N, out, stream)
        nodes_per_step = crr_nodes(N) * n

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
    kernel_ms, vertex_sum = 0.0, 0
    for i in range(args.steps):
        flush_l2(flush)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
        if args.config == 4:
            st = api.tc_last_stats()
            kernel_ms += st["solve_ms"]
            vertex_sum += st["vertex_sum"]
    torch.cuda.synchronize()
    launches = api.launch_count() - launches0
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = max_over_ranks(float(np.sum(step_ms)), pg, dev)
    total_nodes = sum_over_ranks(float(nodes_per_step * args.steps), pg, dev)
    total_opts = sum_over_ranks(float(n * args.steps), pg, dev)
    value = total_nodes / (total_ms / 1e3)

    # roofline of the dominant kernel: FP64 DFMA peak measured on this pool's
    # B200s by tools/fp64_peak.cu (MEASURED_PEAKS.json has no FP64 entry);
    # fallback: the unit-count derivation
    props = torch.cuda.get_device_properties(dev)
    sm_count = props.multi_processor_count
    clk = (clocks or {}).get("sm_max_mhz") or 1965.0
    peak_tflops = sm_count * FP64_LANES_PER_SM * 2 * clk * 1e6 / 1e12
    peak_src = (f"derived: {sm_count} SMs x 64 FP64/clk x 2 x {clk:.0f} MHz "
                "(no FP64 entry in MEASURED_PEAKS.json)")
    fp64_file = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    if os.path.exists(fp64_file):
        try:
            m = json.load(open(fp64_file))
            peak_tflops = float(m["fp64_tflops"])
            peak_src = ("measured: DFMA throughput by tools/fp64_peak.cu on this pool's B200 "
                        "(profiles/r01_fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry)")
        except Exception:
            pass
    if args.config == 4:
        kern_ms = kernel_ms / args.steps
        flop = TC_FLOP_PER_CHILD_VERTEX * 2.0 * vertex_sum / args.steps
        kname = "tc_solve_kernel"
    else:
        # the CRR step is a single kernel launch: its event time is the step time
        kern_ms = float(np.mean(step_ms))
        flop = CRR_FLOP_PER_NODE * nodes_per_step
        kname = "crr_kernel"
    achieved = flop / (kern_ms / 1e3) / 1e12
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved / peak_tflops, "traffic": None, "kernel": kname,
                "kernel_ms_per_step": kern_ms,
                "peak_source": peak_src,
                "flop_model": ("12 flop per child vertex per node-update (DESIGN.md)" if args.config == 4
                               else "6 flop per CRR node-update (DESIGN.md)")}
    if args.config == 4:
        roofline["vertex_sum_per_step"] = vertex_sum / args.steps
        tf = os.path.join(ROOT, "profiles", "r01_traffic_config4.json")
        if os.path.exists(tf):
            try:
                roofline["traffic"] = float(json.load(open(tf))["traffic_bytes_per_step"])
                roofline["traffic_source"] = "ncu dram__bytes_read+write of one step (profiles/r01_traffic_config4.json)"
            except Exception:
                pass

    # end to end through the public C-ABI with HOST buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        pinned = {f: torch.from_numpy(np.ascontiguousarray(getattr(b, f))).pin_memory()
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
                d2h = q.nbytes
            else:
                q = api.price_crr_batch_host(hb, N, stream)
                d2h = q.nbytes
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, pg, dev)
        e2e = {"value": sum_over_ranks(float(nodes_per_step * e2e_steps), pg, dev) / e2e_s,
               "unit": "node-updates/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e2e_steps, "timer": "host wall clock around the synchronous C-ABI call"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, budget_options=args.ref_options)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "node-updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": desc, "N": N, "options_per_gpu": n, "options_total": int(total_opts / args.steps),
                           "options_per_s": total_opts / (total_ms / 1e3),
                           "node_updates_per_option": tc_nodes(N) if args.config == 4 else crr_nodes(N),
                           "l2": "flushed before every timed step (512 MiB write, untimed)",
                           "parallelism": f"dp{world} (independent options per rank, no collective)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks, "step_ms": step_ms}
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
    ap.add_argument("--ref-options", type=int, default=8)
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
