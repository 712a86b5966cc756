"""A/B timing of the light kernels (amtc_debug_set_light_kernel 1 vs 2) on
config-4 subsets and the full config-4 batch (one call each, after warm-up)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(force=os.environ.get("AB_FORCE") == "1"); api.lib()
print(json.dumps({"variant": os.environ.get("AMTC_NVCC_EXTRA", "")}), flush=True)
api.debug_set_split_mode(0)
b = W.config4()
N = 1500
sets = {"puts1184": b.subset(np.nonzero(b.kind == 0)[0][:1184])}
if os.environ.get("AB_ALL", "1") == "1":
    sets["all"] = b
api.price_american_tc_batch(api.device_batch(b.subset(np.arange(4))), 20)
for name, sub in sets.items():
    cols = api.device_batch(sub)
    res = {}
    for mode in (1, 2):
        api.debug_set_light_kernel(mode)
        torch.cuda.synchronize(); t = time.time()
        out, rc = api.price_american_tc_batch(cols, N)
        torch.cuda.synchronize(); dt = time.time() - t
        q = api.quotes_to_numpy(out)
        res[mode] = q
        print(json.dumps({"set": name, "mode": mode, "s": round(dt, 4), "rc": rc, "stats": api.tc_last_stats()}), flush=True)
    d = max(np.max(np.abs(res[1]["ask"] - res[2]["ask"])), np.max(np.abs(res[1]["bid"] - res[2]["bid"])))
    print(json.dumps({"set": name, "max_abs_diff_modes": float(d)}), flush=True)
api.debug_set_light_kernel(1)
