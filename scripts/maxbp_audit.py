"""GPU max_bp (the largest node function held, in vertices) against the oracle's
largest kink count, per config-4 option: the mismatches of the capacity audit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1110_2477_b200 import api, workloads as W
api.lib()
b = W.config4()
z = np.load("tests/golden/oracle_config4_full.npz")
q, rc = api.price_american_tc_batch(api.device_batch(b), 1500)
torch.cuda.synchronize()
q = api.quotes_to_numpy(q)
mk = np.maximum(z["max_kinks_ask"], z["max_kinks_bid"])
d = q["max_bp"] - mk
bad = np.nonzero(np.abs(d) > np.maximum(4, 0.05 * mk))[0]
print("rc", rc, "mismatches", len(bad), "diff range", int(d.min()), int(d.max()))
for i in bad[:20]:
    print(int(i), "kind", int(b.kind[i]), "gpu", int(q["max_bp"][i]), "oracle ask/bid", int(z["max_kinks_ask"][i]), int(z["max_kinks_bid"][i]),
          "k/h", float(b.k[i] / (b.sigma[i] * np.sqrt(b.T[i] / 1500))))
