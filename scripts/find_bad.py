"""Options of the config-4 batch whose GPU status is not OK (or whose prices miss the
oracle), with their parameters; then each re-run alone in every mode."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
b = W.config4()
z = np.load("tests/golden/oracle_config4_full.npz")
q, rc = api.price_american_tc_batch(api.device_batch(b), 1500)
torch.cuda.synchronize()
q = api.quotes_to_numpy(q)
bad = np.nonzero(q["status"] != 0)[0]
print("rc", rc, "bad", bad.tolist())
for i in bad:
    r = b.row(int(i))
    print(json.dumps({k: (float(v) if not isinstance(v, (int, np.integer)) else int(v)) for k, v in r.items()}),
          "oracle", float(z["ask"][i]), float(z["bid"][i]), "maxk", int(z["max_kinks_ask"][i]), int(z["max_kinks_bid"][i]))
sub = b.subset(bad)
for split, full, light in ((0, 0, 1), (0, 1, 1), (0, 0, 0), (1, 0, 1)):
    api.debug_set_split_mode(split); api.debug_set_full_kernel(full); api.debug_set_light_kernel(light)
    qq, rc = api.price_american_tc_batch(api.device_batch(sub), 1500)
    torch.cuda.synchronize()
    qq = api.quotes_to_numpy(qq)
    print("split", split, "full", full, "light", light, "rc", rc, qq["status"].tolist(), qq["ask"].tolist()[:3], qq["bid"].tolist()[:3])
