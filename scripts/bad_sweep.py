"""The eight config-4 calls that the strip kernel reported EUNBOUNDED: per party,
per heavy threshold, which path fails."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
b = W.config4()
bad = [173, 4565, 8068, 8859, 9076, 10837, 12129, 14473]
sub = b.subset(np.array(bad))
api.debug_set_split_mode(0)
for tl in (-1, 16, 32, 128, 512, 4096):
    api.debug_set_heavy_threshold(tl)
    qq, rc = api.price_american_tc_batch(api.device_batch(sub), 1500)
    torch.cuda.synchronize()
    qq = api.quotes_to_numpy(qq)
    print(os.environ.get("AMTC_NVCC_EXTRA", ""), "tl", tl, "rc", rc, qq["status"].tolist(), api.tc_last_stats()["retried_items"], flush=True)
api.debug_set_heavy_threshold(-1)
for N in (200, 400, 800, 1200):
    qq, rc = api.price_american_tc_batch(api.device_batch(sub), N)
    torch.cuda.synchronize()
    print("N", N, "rc", rc, api.quotes_to_numpy(qq)["status"].tolist(), flush=True)
