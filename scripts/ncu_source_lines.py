"""Per-source-line summary of an ncu report captured with --import-source on
(-lineinfo build): warp instructions executed, stall samples and the local /
global memory instructions of each line of the chosen kernel.

  python scripts/ncu_source_lines.py gpurun_out/<rep>.ncu-rep [kernel-substring] [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else "strip_kernel<4"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    # the source page prints one CSV table per kernel, preceded by a header line naming the kernel
    blocks, cur, name = [], [], None
    for ln in text.splitlines():
        if ln.startswith('"') and cur is not None:
            cur.append(ln)
        elif ln.strip() and not ln.startswith('"'):
            if cur:
                blocks.append((name, cur))
            name, cur = ln.strip(), []
    if cur:
        blocks.append((name, cur))
    for name, rows in blocks:
        if want not in (name or ""):
            continue
        rd = list(csv.DictReader(io.StringIO("\n".join(rows))))
        if not rd:
            continue
        cols = rd[0].keys()
        c_src = next((c for c in cols if c.lower().startswith("source") and "sass" not in c.lower()), None)
        c_sass = next((c for c in cols if c.lower() in ("source", "sass")), None)
        c_inst = next((c for c in cols if "Instructions Executed" in c and "Thread" not in c and "Pred" not in c), None)
        c_samp = next((c for c in cols if c.startswith("# Samples") or c == "Warp Stall Sampling (All Samples)"), None)
        c_file = next((c for c in cols if "File" in c or "Address" == c), None)
        print("kernel:", name)
        print("columns:", list(cols)[:40])
        agg = collections.defaultdict(lambda: [0, 0, 0])
        tot_i = tot_s = 0
        for r in rd:
            key = r.get(c_file, "")
            try:
                i = int(float(r.get(c_inst, 0) or 0))
                s = int(float(r.get(c_samp, 0) or 0))
            except ValueError:
                continue
            agg[key][0] += i
            agg[key][1] += s
            sass = r.get(c_sass, "") or ""
            if "LDL" in sass or "STL" in sass:
                agg[key][2] += i
            tot_i += i
            tot_s += s
        print(f"total warp instructions {tot_i}, stall samples {tot_s}")
        for key, (i, s, l) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
            print(f"{s / max(tot_s, 1) * 100:6.2f}% samples  {i / max(tot_i, 1) * 100:6.2f}% inst  local-inst {l / max(tot_i, 1) * 100:5.2f}%  {key}")


if __name__ == "__main__":
    main()
