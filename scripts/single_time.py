"""GPU timing of single-tree TC calls (configs 1, 3, 5b) in split vs whole-tree mode."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
def run(r, N, k, kind, mode):
    api.debug_set_split_mode(mode)
    api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], 40, k, kind)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        q = api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N, k, kind)
        ts.append(time.perf_counter() - t)
    api.debug_set_split_mode(-1)
    return q, 1e3 * min(ts)
c1 = W.config1().row(0)
for mode in (0, 1):
    q, ms = run(c1, 100, c1["k"], 0, mode)
    print(json.dumps({"cfg": 1, "mode": mode, "N": 100, "ms": ms, "q": q}), flush=True)
r3 = dict(S0=100.0, K=100.0, T=1.0, sigma=0.2, R=0.05)
for kind in (0, 1):
    for N in (250, 1000, 2000):
        for k in (0.005, 0.02):
            for mode in ((0, 1) if N == 2000 else (1,)):
                q, ms = run(r3, N, k, kind, mode)
                print(json.dumps({"cfg": 3, "kind": kind, "mode": mode, "N": N, "k": k, "ms": ms, "q": q}), flush=True)
r = W.config5b().row(0)
for mode in (1, 0):
    q, ms = run(r, 8000, r["k"], 0, mode)
    print(json.dumps({"cfg": "5b", "mode": mode, "N": 8000, "ms": ms, "q": q}), flush=True)
