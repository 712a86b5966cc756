"""A/B of the full solvers (amtc_debug_set_full_kernel 1 = amtc_full.cu, 0 =
the strip kernel) on config-4 subsets and the whole batch: one call each after
warm-up, per-kernel times, the max difference between the modes and, for the
options the cached oracle file covers, the max relative error vs the oracle."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(force=os.environ.get("AB_FORCE") == "1"); api.lib()
print(json.dumps({"variant": os.environ.get("AMTC_NVCC_EXTRA", "")}), flush=True)
api.debug_set_split_mode(0)
b = W.config4()
N = 1500
ref = None
for f in ("tests/golden/oracle_config4_full.npz", "tests/golden/oracle_config4_full.npz.partial.npz"):
    if os.path.exists(f):
        z = np.load(f)
        done = z["done"] if "done" in z.files else np.ones(len(b), bool)
        ref = (done, z["ask"], z["bid"])
        break
calls = np.nonzero(b.kind == 1)[0]
bulls = np.nonzero(b.kind == 2)[0]
sets = {"calls512": calls[:512], "bulls512": bulls[:512], "puts1184": np.nonzero(b.kind == 0)[0][:1184]}
if os.environ.get("AB_ALL", "1") == "1":
    sets["all"] = np.arange(len(b))
if os.environ.get("AB_SETS"):
    sets = {k: v for k, v in sets.items() if k in os.environ["AB_SETS"].split(",")}
modes = [int(m) for m in os.environ.get("AB_MODES", "1,0").split(",")]
api.price_american_tc_batch(api.device_batch(b.subset(np.arange(4))), 20)
for name, idx in sets.items():
    cols = api.device_batch(b.subset(idx))
    res = {}
    for mode in modes:
        api.debug_set_full_kernel(mode)
        torch.cuda.synchronize(); t = time.time()
        out, rc = api.price_american_tc_batch(cols, N)
        torch.cuda.synchronize(); dt = time.time() - t
        q = api.quotes_to_numpy(out)
        res[mode] = q
        rec = {"set": name, "mode": mode, "s": round(dt, 4), "rc": rc, "stats": api.tc_last_stats()}
        if ref is not None:
            d = ref[0][idx]
            if d.any():
                for p in ("ask", "bid"):
                    o = ref[1 if p == "ask" else 2][idx][d]
                    g = q[p][d]
                    err = np.abs(g - o) / np.maximum(np.abs(o), 1e-300)
                    floor = 4 * N * 2.220446049250313e-16 * 100.0
                    bad = (np.abs(g - o) > np.maximum(1e-9 * np.abs(o), floor)) | ~np.isfinite(g)
                    rec[p + "_vs_oracle"] = {"n": int(d.sum()), "max_rel": float(np.max(np.where(np.abs(o) > 1e-6, err, 0))),
                                             "bad": int(bad.sum())}
        print(json.dumps(rec), flush=True)
    if len(modes) == 2:
        dd = max(np.nanmax(np.abs(res[modes[0]]["ask"] - res[modes[1]]["ask"])),
                 np.nanmax(np.abs(res[modes[0]]["bid"] - res[modes[1]]["bid"])))
        print(json.dumps({"set": name, "max_abs_diff_modes": float(dd)}), flush=True)
api.debug_set_full_kernel(0)
