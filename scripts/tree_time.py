"""GPU timing of the single large-tree paths (config 5a CRR, config 5b TC)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
r = W.config5a().row(0)
for N in (1000, 10000, 100000, 1000000):
    api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter()
        v = api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N)
        ts.append(time.perf_counter() - t)
    nodes = N * (N + 1) / 2
    print(json.dumps({"cfg": "5a", "N": N, "price": v, "ms": 1e3 * min(ts), "node_updates_per_s": nodes / min(ts)}), flush=True)
r = W.config5b().row(0)
for N in (1000, 8000) if len(sys.argv) < 2 else ():
    t = time.perf_counter()
    q = api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, r["k"], 0)
    dt = time.perf_counter() - t
    print(json.dumps({"cfg": "5b", "N": N, "q": q, "ms": 1e3 * dt}), flush=True)
