"""One small solver invocation for compute-sanitizer runs (scripts/gpu_sanitize.sh).
usage: sanitize_case.py whole|split|concurrent|retry|strip|crr|tree"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1110_2477_b200 import api, workloads as W

case = sys.argv[1]
api.lib()
b = W.config4()
N = int(os.environ.get("SAN_N", "96"))
# a few calls (heavy buyers: tier 3 work sharing), bull spreads and puts
idx = np.concatenate([np.nonzero(b.kind == 1)[0][:6], np.nonzero(b.kind == 2)[0][:3], np.nonzero(b.kind == 0)[0][:3]])
sub = b.subset(idx)
if case == "whole":       # whole-tree mode, everything on amtc_full.cu
    api.debug_set_split_mode(0); api.debug_set_light_kernel(0); api.debug_set_full_kernel(1)
    api.debug_set_heavy_threshold(8)
elif case == "split":     # strip-split mode (progress counters in global memory)
    api.debug_set_split_mode(1)
elif case == "concurrent":  # light kernel on a second stream beside the full kernel
    api.debug_set_split_mode(0); api.debug_set_light_kernel(1); api.debug_set_heavy_threshold(8)
elif case == "retry":     # shrunken arenas: capacity retry passes
    api.debug_set_split_mode(0); api.debug_set_arena_shift(12); api.debug_set_heavy_threshold(8)
elif case == "strip":     # the round-1 strip kernel as the full solver
    api.debug_set_split_mode(0); api.debug_set_full_kernel(0); api.debug_set_heavy_threshold(8)
if case == "crr":
    p = api.price_crr_batch_host(W.config2().subset(np.arange(64)), 200)
    print("crr ok", float(np.nanmax(p)))
    p = api.price_crr_batch_host(W.config2().subset(np.arange(8)), 1300)  # the strip kernel (N > 1152)
    print("crr strip ok", float(np.nanmax(p)))
elif case == "tree":
    print("tree", api.price_crr_tree(100.0, 100.0, 1.0, 0.3, 0.05, 3000, api.PUT))
else:
    q, rc = api.price_american_tc_batch_host(sub, N)
    print(case, "rc", rc, "stats", api.tc_last_stats(), "finite", bool(np.isfinite(q["ask"]).all()))
