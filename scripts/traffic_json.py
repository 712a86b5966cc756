"""DRAM traffic of one config-4 step's solver kernels from an ncu report
(dram__bytes_read.sum + dram__bytes_write.sum per launch), written to
profiles/r02_traffic_config4.json for bench.py's roofline.traffic.

  python scripts/traffic_json.py gpurun_out/<report>.ncu-rep  (or a --csv --page raw export)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(path):
    if path.endswith(".csv"):
        text = open(path).read()
    else:
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base", "--metrics",
                               "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                              capture_output=True, text=True, check=True).stdout
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def val(r, key):
    for k, v in r.items():
        if k.startswith(key):
            try:
                return float(str(v).replace(",", ""))
            except ValueError:
                return None
    return None


def main():
    rs = [r for r in rows(sys.argv[1]) if val(r, "dram__bytes_read.sum") is not None]  # (skips the units row)
    out = {"what": "dram__bytes_read.sum + dram__bytes_write.sum per launch of one config-4 step's solver kernels "
                   "(ncu --clock-control none on bench.py --steps 1 --warmup 1; the benched code)",
           "source": os.path.basename(sys.argv[1]), "kernels": []}
    for r in rs:
        name = r.get("Kernel Name", "?")
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        out["kernels"].append({"kernel": name, "read": rd, "write": wr, "ns": val(r, "gpu__time_duration.sum")})
    # --print-units base: bytes and nanoseconds
    full = [k for k in out["kernels"] if "strip_kernel" in k["kernel"] or "full_kernel" in k["kernel"]]
    light = [k for k in out["kernels"] if "light_kernel" in k["kernel"]]
    if full:
        out["full_kernel_bytes"] = full[-1]["read"] + full[-1]["write"]
        out["full_kernel"] = full[-1]["kernel"]
    if light:
        out["light_kernel_bytes"] = light[-1]["read"] + light[-1]["write"]
    path = os.path.join(ROOT, "profiles", "r02_traffic_config4.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}))


if __name__ == "__main__":
    main()
