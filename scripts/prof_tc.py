"""GPU profiling helper: one batched TC call on a subset of config 4.
usage: prof_tc.py KIND|all N_OPTIONS N [party_filter]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
if os.environ.get("AMTC_LIGHT") == "0": api.debug_set_light_kernel(False)
if os.environ.get("AMTC_SPLIT") is not None: api.debug_set_split_mode(int(os.environ["AMTC_SPLIT"]))
kind = sys.argv[1]; n = int(sys.argv[2]); N = int(sys.argv[3])
b = W.config4()
idx = np.arange(len(b)) if kind == "all" else np.nonzero(b.kind == int(kind))[0]
sub = b.subset(idx[:n])
# warm-up on a tiny batch (module load, workspace)
api.price_american_tc_batch(api.device_batch(b.subset(idx[:2])), 20)
cols = api.device_batch(sub)
torch.cuda.synchronize()
t = time.time()
out, rc = api.price_american_tc_batch(cols, N)
torch.cuda.synchronize()
dt = time.time() - t
q = api.quotes_to_numpy(out)
print(json.dumps({"kind": kind, "n": len(sub), "N": N, "s": round(dt, 4), "rc": rc, "stats": api.tc_last_stats(),
                  "max_bp": int(q["max_bp"].max()), "node_updates_per_s": len(sub) * (N + 1) * (N + 2) / 2 / dt}))
