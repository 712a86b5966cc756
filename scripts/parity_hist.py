"""Error distribution of the CUDA path against the cached full-batch oracle
files (configs 4 and 2; A19): histograms of the relative error
|g - o| / |o| and of the absolute error in units of N eps S0, and how many
comparisons the rounding floor decided.  Writes profiles/r02_parity_error_hist.json.

  python scripts/parity_hist.py            (GPU)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1110_2477_b200 import api, workloads as W  # noqa: E402
from tolerance import check_arrays  # noqa: E402

EPS = float(np.finfo(np.float64).eps)


def hist(g, o, N, S0):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    err = np.abs(g - o)
    nz = o != 0
    rel = np.where(nz, err / np.where(nz, np.abs(o), 1.0), np.inf)
    units = err / (N * EPS * np.asarray(S0, np.float64))
    rb = [0, 1e-15, 1e-14, 1e-13, 1e-12, 1e-11, 1e-10, 1e-9, 1e-8, 1e-7, np.inf]
    ub = [0, 0.01, 0.1, 0.5, 1, 2, 4, 8, 16, np.inf]
    ok, floor_used = check_arrays(g, o, N, S0)
    return {
        "n": int(o.size), "pass": int(ok.sum()), "floor_used": int(floor_used),
        "exact_zero_refs": int((~nz).sum()), "bitwise_equal": int((g == o).sum()),
        "max_rel_err_nonzero_refs": float(rel[nz].max()) if nz.any() else 0.0,
        "max_err_in_N_eps_S0": float(units.max()),
        "rel_err_hist": {f"<{b:g}": int(((rel >= a) & (rel < b)).sum()) for a, b in zip(rb[:-1], rb[1:])},
        "abs_err_hist_N_eps_S0": {f"<{b:g}": int(((units >= a) & (units < b)).sum()) for a, b in zip(ub[:-1], ub[1:])},
        "floor_cases": [{"ref": float(o[i]), "gpu": float(g[i]), "err_in_N_eps_S0": float(units[i])}
                        for i in np.nonzero(ok & ~(err <= 1e-9 * np.abs(o)))[0][:20]],
    }


def main():
    api.lib()
    out = {"tolerance": "tests/tolerance.py (A19): |g-o| <= 1e-9 |o| or <= 4 N eps S0",
           "source": "scripts/parity_hist.py: CUDA path (bench launch configuration) vs tests/golden/oracle_config*_full.npz"}
    b = W.config4()
    z = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config4_full.npz"))
    assert str(z["sha256"]) == W.soa_sha256(b)
    q, rc = api.price_american_tc_batch(api.device_batch(b), W.CONFIG4_N)
    torch.cuda.synchronize()
    q = api.quotes_to_numpy(q)
    out["config4"] = {"N": W.CONFIG4_N, "rc": int(rc),
                      "ask": hist(q["ask"], z["ask"], W.CONFIG4_N, b.S0),
                      "bid": hist(q["bid"], z["bid"], W.CONFIG4_N, b.S0)}
    b2 = W.config2()
    z2 = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2_full.npz"))
    assert str(z2["sha256"]) == W.soa_sha256(b2)
    p = api.price_crr_batch(api.device_batch(b2), W.CONFIG2_N)
    torch.cuda.synchronize()
    out["config2"] = {"N": W.CONFIG2_N, "price": hist(p.cpu().numpy(), z2["price"], W.CONFIG2_N, b2.S0)}
    path = os.environ.get("PH_OUT") or os.path.join(ROOT, "profiles", "r02_parity_error_hist.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: (v if k not in ("config4", "config2") else
                          {p_: {kk: vv for kk, vv in v[p_].items() if kk in ("n", "pass", "floor_used",
                                "max_rel_err_nonzero_refs", "max_err_in_N_eps_S0")} for p_ in v if p_ != "N" and p_ != "rc"})
                      for k, v in out.items()}))


if __name__ == "__main__":
    main()
