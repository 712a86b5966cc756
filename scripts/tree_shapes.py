"""GPU timing of the k = 0 single-tree sweep shapes (amtc_debug_set_tree_shape):
1 one launch per band, 2..5 the wavefront kernel.  One JSON line per (shape, N)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
r = W.config5a().row(0)
Ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [10000, 100000, 1000000]
SHAPES = [int(x) for x in os.environ.get('TS_SHAPES', '1,2,3,4,5,0').split(',')]
for shape in SHAPES:
    api.debug_set_tree_shape(shape)
    for N in Ns:
        api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(); t = time.perf_counter()
            v = api.price_crr_tree(r["S0"], r["K"], r["T"], r["sigma"], r["R"], N)
            ts.append(time.perf_counter() - t)
        print(json.dumps({"shape": shape, "N": N, "price": v, "ms_min": 1e3 * min(ts),
                          "ms_med": 1e3 * sorted(ts)[2]}), flush=True)
api.debug_set_tree_shape(0)
