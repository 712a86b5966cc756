"""Full-batch oracle references for the headline configs ("Reference
outputs precomputed once on all cores of this container (hash-keyed) ... Parity
checks all 16,384 against the cached file").

Calls ONLY oracle/ (and the seeded generators in paper_1110_2477_b200/workloads.py,
which hold none of the method's arithmetic).  Never reads the CUDA path.

  python scripts/make_full_refs.py config4 [threads]   # ~2 h on 8 cores
  python scripts/make_full_refs.py config2 [threads]   # a few minutes

Writes tests/golden/oracle_<cfg>_full.npz keyed by workloads.soa_sha256(batch).
config4 also stores the oracle's SURVEY 8(d) cost-model counts per option and the
batch's per-level kink statistics (oracle.new_level_stats layout, summed over
options).  Progress is checkpointed to <file>.partial.npz so an interrupted run
resumes where it stopped.
"""
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor, as_completed

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_1110_2477_b200 import workloads as W  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
TC_FIELDS = ("ask", "bid", "status", "max_kinks_ask", "max_kinks_bid", "sum_kinks_ask",
             "sum_kinks_bid", "crossings", "fp64_ops", "merge_visits", "restrict_cvx",
             "restrict_ncvx", "scale_visits", "fp64_ops_ask", "fp64_ops_bid", "seconds")


def opt(row):
    return O.Option(row["S0"], row["K"], row["T"], row["sigma"], row["R"], row["k"], row["kind"], row["K2"])


def config4(threads):
    b = W.config4()
    N = W.CONFIG4_N
    n = len(b)
    path = os.path.join(GOLD, "oracle_config4_full.npz")
    part = path + ".partial.npz"
    res = {f: np.full(n, np.nan) for f in TC_FIELDS}
    done = np.zeros(n, dtype=bool)
    lvl = O.new_level_stats(N)
    if os.path.exists(part):
        z = np.load(part)
        assert str(z["sha256"]) == W.soa_sha256(b)
        done = z["done"].copy()
        for f in TC_FIELDS:
            res[f] = z[f].copy()
        lvl = z["level_stats"].copy()
        print("resuming:", int(done.sum()), "done", flush=True)
    # heaviest first (calls / bull spreads at large k/h carry the buyer's sawtooth,
    # DESIGN.md 5) so the tail of the run is short
    h = b.sigma * np.sqrt(b.T / N)
    est = (1.0 + 8.0 * (b.kind != W.PUT)) * (1.0 + b.k / h)
    order = [int(i) for i in np.argsort(-est) if not done[i]]
    lock = threading.Lock()
    local = threading.local()
    accs = []

    def run(i):
        if not hasattr(local, "acc"):
            local.acc = O.new_level_stats(N)
            with lock:
                accs.append(local.acc)
        t = time.time()
        q = O.price_tc(opt(b.row(i)), N, level_stats=local.acc)
        return i, q, time.time() - t

    def save(final=False):
        tot = lvl.copy()
        for a in accs:
            tot += a
        out = dict(sha256=W.soa_sha256(b), N=N, done=done, level_stats=tot,
                   source="oracle/amtc_oracle.c via scripts/make_full_refs.py (BASELINE.json config 4, all options)",
                   **res)
        np.savez_compressed((path if final else part) + ".tmp.npz", **out)
        os.replace((path if final else part) + ".tmp.npz", path if final else part)

    t0 = time.time()
    last = t0
    with ThreadPoolExecutor(threads) as ex:
        futs = [ex.submit(run, i) for i in order]
        for k, fu in enumerate(as_completed(futs)):
            i, q, sec = fu.result()
            for f in TC_FIELDS:
                res[f][i] = sec if f == "seconds" else getattr(q, f)
            done[i] = True
            if time.time() - last > 120:
                with lock:
                    save()
                last = time.time()
                print(f"{int(done.sum())}/{n} after {time.time() - t0:.0f} s", flush=True)
    save(final=True)
    if os.path.exists(part):
        os.remove(part)


def config2(threads):
    b = W.config2()
    N = W.CONFIG2_N
    rows = [opt(b.row(i)) for i in range(len(b))]
    price = np.array(O.price_crr_many(rows, N, threads=threads))
    path = os.path.join(GOLD, "oracle_config2_full.npz")
    np.savez_compressed(path, sha256=W.soa_sha256(b), N=N, price=price,
                        source="oracle/amtc_oracle.c via scripts/make_full_refs.py (BASELINE.json config 2, all options)")


if __name__ == "__main__":
    what = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else len(os.sched_getaffinity(0))
    t = time.time()
    {"config4": config4, "config2": config2}[what](threads)
    print(what, "done in", round(time.time() - t, 1), "s", flush=True)
