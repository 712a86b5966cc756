"""GPU diagnostic: time TC batches by option class (puts / calls / bulls) and the full config 4."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W, build
build.build(); api.lib()
b = W.config4()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 1024]
for kind in (0, 1, 2):
    idx = np.nonzero(b.kind == kind)[0]
    for m in sizes:
        sub = b.subset(idx[:m])
        cols = api.device_batch(sub)
        torch.cuda.synchronize()
        t = time.time()
        out, rc = api.price_american_tc_batch(cols, N)
        torch.cuda.synchronize()
        dt = time.time() - t
        q = api.quotes_to_numpy(out)
        print(json.dumps({"kind": kind, "n": m, "N": N, "s": round(dt, 3), "rc": rc, "stats": api.tc_last_stats(),
                          "max_bp": int(q["max_bp"].max()), "opt_per_s": m / dt}), flush=True)
