"""Phase counters of the full solver (build with AMTC_NVCC_EXTRA=-DAMTC_F_PROF=1):
python scripts/prof_full.py [set ...]   sets: all calls512 bulls512 callsK (K = count)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(force=os.environ.get("PF_FORCE") == "1"); api.lib()
api.debug_set_split_mode(0)
if os.environ.get("PF_LIGHT") is not None: api.debug_set_light_kernel(int(os.environ["PF_LIGHT"]))
b = W.config4()
N = 1500
api.price_american_tc_batch(api.device_batch(b.subset(np.arange(4))), 20)
for name in (sys.argv[1:] or ["all"]):
    if name == "all": idx = np.arange(len(b))
    elif name.startswith("calls"): idx = np.nonzero(b.kind == 1)[0][: int(name[5:])]
    elif name.startswith("bulls"): idx = np.nonzero(b.kind == 2)[0][: int(name[5:])]
    cols = api.device_batch(b.subset(idx))
    api.debug_full_profile(reset=True)
    torch.cuda.synchronize(); t = time.time()
    out, rc = api.price_american_tc_batch(cols, N)
    torch.cuda.synchronize(); dt = time.time() - t
    p = api.debug_full_profile(reset=True)
    rec = {"set": name, "s": round(dt, 4), "rc": rc, "stats": api.tc_last_stats(), "prof": p}
    if p and p["total_cycles"]:
        T = p["total_cycles"]
        rec["frac"] = {k: round(p[k] / T, 4) for k in ("heavy_cycles", "wait_cycles", "idle_cycles", "tier2_cycles")}
        rec["cycles_per_served"] = p["heavy_cycles"] / max(p["served"], 1)
    print(json.dumps(rec), flush=True)
