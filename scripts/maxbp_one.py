import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
b = W.config4()
sub = b.subset(np.array([96, 252, 256, 542]))
for split, full, light in ((0, 0, 1), (0, 1, 1), (0, 0, 0), (0, 0, 2)):
    api.debug_set_split_mode(split); api.debug_set_full_kernel(full); api.debug_set_light_kernel(light)
    q, rc = api.price_american_tc_batch(api.device_batch(sub), 1500)
    torch.cuda.synchronize()
    q = api.quotes_to_numpy(q)
    print(split, full, light, rc, q["max_bp"].tolist(), q["ask"].tolist())
for i in (96, 252):
    r = b.row(i)
    for kind in (api.CALL,):
        print(i, api.price_american_tc(r["S0"], r["K"], r["T"], r["sigma"], r["R"], 1500, r["k"], kind))
