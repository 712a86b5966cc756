"""Summary of an ncu --set full report (one config-4 step's solver kernels) for
profiles/: time, DRAM bytes, FP64-pipe utilisation, issue, occupancy, local
(spill) traffic and cache hit rates per kernel.

  python scripts/ncu_summary.py gpurun_out/<report>.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration [ns]"),
    ("dram__bytes_read.sum", "DRAM read [B]"),
    ("dram__bytes_write.sum", "DRAM write [B]"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst / peak [%]"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active cycles [%]"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_fp64.sum", "FP64-pipe warp instructions"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "instruction throughput [% peak]"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy [%]"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy [%]"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic shared / CTA [B]"),
    ("l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "local (spill) loads [B]"),
    ("l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum", "local (spill) stores [B]"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate [%]"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate [%]"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio", "long-scoreboard stall / issue"),
]


def main():
    rep = sys.argv[1]
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                          capture_output=True, text=True, check=True).stdout
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    data = rows[1:]  # rows[0] holds the units
    print(f"ncu --set full report {rep.split('/')[-1]} (--clock-control none); one config-4 step, bench.py --steps 1 --warmup 1")
    for r in data:
        name = r.get("Kernel Name", "?")
        print(f"\n== {name}  grid {r.get('Grid Size', '?')} block {r.get('Block Size', '?')}")
        for key, label in METRICS:
            v = r.get(key)
            if v in (None, ""):
                continue
            print(f"  {label:36s} {v}")
        try:
            ins = float(str(r.get("smsp__inst_executed.sum", "0")).replace(",", ""))
            f64 = float(str(r.get("sm__inst_executed_pipe_fp64.sum", "0")).replace(",", ""))
            if ins:
                print(f"  {'FP64-pipe share of instructions':36s} {f64 / ins:.4f}")
        except ValueError:
            pass


if __name__ == "__main__":
    main()
