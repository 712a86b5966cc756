"""Write oracle reference values for the GPU parity tests (tests/golden/).

Calls ONLY oracle/ (and the seeded generators in paper_1110_2477_b200/workloads.py,
which hold none of the method's arithmetic).  Never reads the CUDA path.
Usage: python scripts/make_oracle_refs.py [config2|config3|config4|config5b|all]
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_1110_2477_b200 import workloads as W  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
THREADS = len(os.sched_getaffinity(0))


def opt(row):
    return O.Option(row["S0"], row["K"], row["T"], row["sigma"], row["R"], row["k"], row["kind"], row["K2"])


def config3():
    pts = W.config3()

    def run(p):
        b, N = p
        r = b.row(0)
        t = time.time()
        q = O.price_tc(opt(r), N)
        return dict(kind=r["kind"], k=r["k"], N=N, ask=q.ask, bid=q.bid, status=q.status,
                    max_kinks=max(q.max_kinks_ask, q.max_kinks_bid), seconds=time.time() - t)

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(run, sorted(pts, key=lambda p: -p[1])))
    return {"_source": "oracle/amtc_oracle.c via scripts/make_oracle_refs.py (BASELINE.json config 3)",
            "points": res}


def config4(n_sample=64, seed=7):
    b = W.config4()
    idx = np.sort(np.random.default_rng(seed).choice(len(b), n_sample, replace=False))

    def run(i):
        r = b.row(int(i))
        q = O.price_tc(opt(r), W.CONFIG4_N)
        return dict(index=int(i), ask=q.ask, bid=q.bid, status=q.status,
                    max_kinks=max(q.max_kinks_ask, q.max_kinks_bid))

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(run, idx))
    return {"_source": "oracle/amtc_oracle.c via scripts/make_oracle_refs.py (BASELINE.json config 4, "
                       f"seeded sample: numpy default_rng({seed}).choice(16384, {n_sample}))",
            "N": W.CONFIG4_N, "samples": res}


def config2(n_sample=256, seed=11):
    b = W.config2()
    idx = np.sort(np.random.default_rng(seed).choice(len(b), n_sample, replace=False))

    def run(i):
        r = b.row(int(i))
        return dict(index=int(i), price=O.price_crr(opt(r), W.CONFIG2_N))

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(run, idx))
    return {"_source": "oracle/amtc_oracle.c via scripts/make_oracle_refs.py (BASELINE.json config 2, "
                       f"seeded sample: numpy default_rng({seed}).choice(65536, {n_sample}))",
            "N": W.CONFIG2_N, "samples": res}


def config5b():
    r = W.config5b().row(0)
    t = time.time()
    q = O.price_tc(opt(r), W.CONFIG5B_N)
    return {"_source": "oracle/amtc_oracle.c via scripts/make_oracle_refs.py (BASELINE.json config 5b)",
            "N": W.CONFIG5B_N, "ask": q.ask, "bid": q.bid, "status": q.status,
            "max_kinks": max(q.max_kinks_ask, q.max_kinks_bid), "seconds": time.time() - t}


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("config2", config2), ("config4", config4), ("config3", config3), ("config5b", config5b)):
        if what not in (name, "all"):
            continue
        t = time.time()
        data = fn()
        with open(os.path.join(GOLD, f"oracle_{name}.json"), "w") as f:
            json.dump(data, f, indent=1)
        print(name, "done in", round(time.time() - t, 1), "s", flush=True)
