"""Per-function / per-source-line summary of an ncu report that holds the
SourceCounters section of strip_kernel<4,4,20> (warp stall samples and executed
instructions per SASS instruction).  The SASS addresses are mapped to source
lines through nvdisasm's line table of a local -lineinfo build of the same
sources (ncu's own CUDA view lists only the kernel's file, not the inlined
headers).

  python scripts/ncu_source_lines.py gpurun_out/<rep>.ncu-rep > profiles/<name>.txt
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FUNCS = ("node_update_block", "node_update_chunk", "node_updateE", "root_min", "tc_root", "serve_one", "div_rn", "dsqrt")


def line_table():
    """offset -> (function, (file, line), sass) for the strip_kernel<4,4,20,...> section"""
    sys.path.insert(0, ROOT)
    from paper_1110_2477_b200 import build as B
    tmp = tempfile.mkdtemp()
    obj = os.path.join(tmp, "strip.o")
    subprocess.run([B.NVCC, *B.FLAGS, "-c", os.path.join(B.CSRC, "amtc_strip.cu"), "-o", obj], check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=tmp, check=True, stdout=subprocess.DEVNULL)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], cwd=tmp, capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(dis) if l.startswith("_ZN4amtc12strip_kernelILi4ELi4ELi20")][0]
    cur, fn, omap = None, "kernel body", {}
    for l in dis[start:]:
        if l.startswith("_ZN4amtc12strip_kernelILi") and "Li4ELi4ELi20" not in l:
            break
        if l.strip().startswith(".section") and omap:
            break
        m = re.match(r"\$_ZN4amtc12strip_kernel\S*?\$(\S+):", l)
        if m:
            for key in FUNCS:
                if key in m.group(1):
                    fn = key
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);", l)
        if m:
            omap[int(m.group(1), 16)] = (fn, cur, m.group(2))
    return omap


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    omap = line_table()
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    best = None
    for b in text.split('"Kernel Name"')[1:]:
        rd = list(csv.DictReader(io.StringIO("\n".join(b.split("\n")[1:]))))
        tot = sum(int(r["Instructions Executed"] or 0) for r in rd)
        if best is None or tot > best[0]:
            best = (tot, rd, b.split("\n")[0])
    tot, rd, name = best
    base = int(rd[0]["Address"], 16)
    stall_cols = [c for c in rd[0].keys() if c.startswith("stall_") and "Not Issued" not in c]
    byfn = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    byline = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    allst = collections.Counter()
    tots = 0
    for r in rd:
        m = omap.get(int(r["Address"], 16) - base)
        i = int(r["Instructions Executed"] or 0)
        s = int(r["# Samples"] or 0)
        tots += s
        for c in stall_cols:
            allst[c] += int(r[c] or 0)
        if not m:
            continue
        f, ln, _ = m
        for d, k in ((byfn, f), (byline, (f, ln))):
            d[k][0] += i
            d[k][1] += s
            for c in stall_cols:
                v = int(r[c] or 0)
                if v:
                    d[k][2][c] += v
    print(f"report {os.path.basename(rep)}; kernel{name.strip(',')}")
    print(f"static SASS instructions {len(rd)} ({len(rd) * 16 // 1024} KB), warp instructions executed {tot}, stall samples {tots}")
    ssum = sum(allst.values())
    print("stall reasons, all samples [%]:", ", ".join(f"{k[6:]} {v / ssum * 100:.1f}" for k, v in allst.most_common(8)))
    print("\nby function (share of executed warp instructions, of stall samples, top stall reasons in % of its samples)")
    for k, (i, s, st) in sorted(byfn.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:20s} inst {i / tot * 100:5.1f}%  samples {s / tots * 100:5.1f}%  ",
              ", ".join(f"{a[6:]} {b / max(s, 1) * 100:.0f}" for a, b in st.most_common(4)))
    print(f"\ntop {top} source lines by stall samples")
    for k, (i, s, st) in sorted(byline.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"  {k[0]:18s} {k[1][0]}:{k[1][1]:<5d} inst {i / tot * 100:5.2f}%  samples {s / tots * 100:5.2f}%  ",
              ", ".join(f"{a[6:]} {b / max(s, 1) * 100:.0f}" for a, b in st.most_common(3)))


if __name__ == "__main__":
    main()
