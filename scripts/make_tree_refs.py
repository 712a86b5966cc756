"""Oracle values of single large k=0 trees (N >= 2e5) for
tests/test_gpu_tree.py -- the GPU's band kernel at N far beyond what the test
suite can run the oracle on.  Calls ONLY oracle/ (price_crr, the plain scalar
CRR induction of P:79 / P:487).  The appendix put (13.906).

  python scripts/make_tree_refs.py N [N ...]     # ~N^2 / 5.6e7 s each on one core
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_1110_2477_b200 import workloads as W  # noqa: E402


def main():
    a = W.appendix_put().row(0)
    for N in (int(x) for x in sys.argv[1:]):
        t = time.time()
        v = O.price_crr(O.Option(a["S0"], a["K"], a["T"], a["sigma"], a["R"], 0.0, O.PUT), N)
        path = os.path.join(ROOT, "tests", "golden", f"oracle_tree_appendix_put_N{N}.json")
        json.dump({"_source": "oracle/amtc_oracle.c price_crr via scripts/make_tree_refs.py (P:487-489 appendix put)",
                   "S0": a["S0"], "K": a["K"], "T": a["T"], "sigma": a["sigma"], "R": a["R"], "kind": "put",
                   "N": N, "price": v, "seconds": time.time() - t}, open(path, "w"), indent=1)
        print(N, v, round(time.time() - t, 1), flush=True)


if __name__ == "__main__":
    main()
