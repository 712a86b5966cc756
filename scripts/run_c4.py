"""One config-4 batch through the device C-ABI (for ncu captures): python scripts/run_c4.py [full_kernel_mode] [n_options]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
api.debug_set_full_kernel(mode)
api.debug_set_split_mode(0)
b = W.config4()
api.price_american_tc_batch(api.device_batch(b.subset(np.arange(4))), 20)
cols = api.device_batch(b.subset(np.arange(n)))
out, rc = api.price_american_tc_batch(cols, 1500)
torch.cuda.synchronize()
print("rc", rc, api.tc_last_stats())
