"""Per-level latency of ONE warp (no other work on the GPU): a single put item
pair (ask + bid) in whole-tree mode on the light kernel and on the strip kernel."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
api.debug_set_split_mode(0)
b = W.config4()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
sub = b.subset(np.nonzero(b.kind == 0)[0][:1])
cols = api.device_batch(sub)
api.price_american_tc_batch(cols, 50)
for light in (1, 0):
    api.debug_set_light_kernel(light)
    torch.cuda.synchronize(); t = time.time()
    out, rc = api.price_american_tc_batch(cols, N)
    torch.cuda.synchronize(); dt = time.time() - t
    steps = sum(N - 32 * s + 1 for s in range(N // 32 + 1))  # level steps of one item
    print(json.dumps({"light_kernel": light, "N": N, "s": dt, "stats": api.tc_last_stats(),
                      "us_per_level_step": 1e6 * dt / steps}))
api.debug_set_light_kernel(1)
