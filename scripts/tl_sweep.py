"""GPU experiment: time heavy-prone items (config-4 calls) at several tier-3 thresholds."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
b = W.config4()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = 1500
idx = np.nonzero(b.kind == 1)[0][:n]
sub = b.subset(idx)
api.price_american_tc_batch(api.device_batch(b.subset(idx[:2])), 20)
cols = api.device_batch(sub)
ref = None
for tl in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,32,16,8,128").split(",")]:
    api.debug_set_heavy_threshold(tl)
    torch.cuda.synchronize(); t = time.time()
    out, rc = api.price_american_tc_batch(cols, N)
    torch.cuda.synchronize(); dt = time.time() - t
    q = api.quotes_to_numpy(out)
    if ref is None: ref = q
    dd = np.abs(q["bid"] - ref["bid"]) - (1e-9 * np.abs(ref["bid"]) + 1e-10)
    i = int(np.argmax(dd))
    d = {"worst_excess_over_tol": float(dd[i]), "i": i, "bid": float(q["bid"][i]), "ref": float(ref["bid"][i]),
         "max_abs_ask": float(np.max(np.abs(q["ask"] - ref["ask"])))}
    print(json.dumps({"tl": tl, "n": n, "s": round(dt, 4), "rc": rc, "stats": api.tc_last_stats(),
                      "max_bp": int(q["max_bp"].max()), "max_rel_vs_first": d}), flush=True)
api.debug_set_heavy_threshold(0)
