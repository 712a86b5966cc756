"""GPU diagnostic: capacity retry passes per option kind in the config-4 batch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, build, workloads as W
build.build(); api.lib()
b = W.config4()
for name, idx in (("all", np.arange(len(b))), ("puts", np.nonzero(b.kind == 0)[0]),
                  ("calls", np.nonzero(b.kind == 1)[0]), ("bulls", np.nonzero(b.kind == 2)[0])):
    sub = b.subset(idx)
    cols = api.device_batch(sub)
    torch.cuda.synchronize()
    out, rc = api.price_american_tc_batch(cols, W.CONFIG4_N)
    st = api.tc_last_stats()
    print(json.dumps({"set": name, "n": len(sub), "rc": rc, **st}), flush=True)
