"""GPU debug helper: a few TC options at small N through the C-ABI vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
b = W.random_small(n, seed=11, k_max=0.05)
got, rc = api.price_american_tc_batch_host(b, N)
print("rc", rc, "stats", api.tc_last_stats())
worst = 0.0
for i in range(len(b)):
    r = b.row(i)
    q = O.price_tc(O.Option(r["S0"], r["K"], r["T"], r["sigma"], r["R"], r["k"], r["kind"], r["K2"]), N)
    e = max(abs(got["ask"][i] - q.ask), abs(got["bid"][i] - q.bid))
    worst = max(worst, e)
    if e > 1e-9 * max(abs(q.ask), 1) or got["status"][i] != q.status:
        print("MISMATCH", i, r["kind"], got[i], q.ask, q.bid, q.status)
print("N", N, "n", n, "worst abs err", worst)
