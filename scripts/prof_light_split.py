"""Split-mode counters of the light kernel (build with AMTC_NVCC_EXTRA=-DAMTC_L2_PROF=1):
per strip-level, the cycles in the level loop and in blocking waits for the strip to the
right, on config 5b (one put tree, N=8000) and on 8 config-4 puts at N=1500."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
api.debug_set_split_mode(1)
cases = [("5b", W.config5b(), W.CONFIG5B_N), ("puts8", W.config4().subset(np.nonzero(W.config4().kind == 0)[0][:8]), 1500)]
for name, b, N in cases:
    cols = api.device_batch(b)
    api.price_american_tc_batch(cols, N)
    api.debug_full_profile(reset=True)
    torch.cuda.synchronize(); t = time.time()
    q, rc = api.price_american_tc_batch(cols, N)
    torch.cuda.synchronize(); dt = time.time() - t
    out = np.zeros(8, dtype=np.uint64)
    api.lib().amtc_debug_full_profile(out.ctypes.data, 1)
    loop, wait, nw, lv, ne = (int(x) for x in out[:5])
    print(name, "s", round(dt, 4), "rc", rc, "levels", lv, "cycles/level", round(loop / max(lv, 1), 1),
          "wait cycles/level", round(wait / max(lv, 1), 1), "blocking waits", nw, "staged early", ne)
