#!/bin/bash
# session 6 final validation of the rolled-scan build: full GPU suite, smoke, parity histogram, benches of every
# config, launch list, per-kernel counters of one config-4 step; then same-box A/B builds of the code-size options
mkdir -p gpurun_out
T=${1:-s6h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$T.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$T.log
PH_OUT=gpurun_out/r02_parity_error_hist.json timeout 600 python scripts/parity_hist.py > gpurun_out/parity_$T.log 2>&1; echo parity rc=$?; tail -c 600 gpurun_out/parity_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>gpurun_out/bench_$T.err; echo bench rc=$?; tail -c 1200 gpurun_out/bench_$T.log
for c in 2 5 3 1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_c${c}_$T.log 2>&1; echo bench$c rc=$?; done
rm -f gpurun_out/slices_$T.jsonl
for g in 0 3 7; do timeout 300 python bench.py --slice $g/8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/slices_$T.jsonl 2>>gpurun_out/slices_$T.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu-launches rc=$?
timeout 1500 ncu --clock-control none -k regex:"strip_kernel|light_kernel" -s 2 -c 2 \
   --section LaunchStats --section Occupancy \
   --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
   -o gpurun_out/${T}_step -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$T.log 2>&1; echo ncu-step rc=$?
run() {
  name=$1; shift
  AMTC_NVCC_EXTRA="$*" timeout 900 python -m paper_1110_2477_b200.build --force > gpurun_out/build_${T}_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/build_${T}_$name.log; return; }
  timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_$name.log 2>&1
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${T}_$name.log").read().strip().splitlines()[-1])
p = d["parity"]
print("$name", [round(x, 1) for x in d["step_ms"]], "ask", p["ask"]["pass"], p["ask"]["fail"], "bid", p["bid"]["pass"], p["bid"]["fail"], flush=True)
PY
}
run scans_only -DAMTC_NO_LANE_MERGED -DAMTC_NO_ENTRY_KNOWN -DAMTC_UNROLLED_RANK
run all_unrolled -DAMTC_UNROLLED_SCANS -DAMTC_NO_LANE_MERGED -DAMTC_NO_ENTRY_KNOWN -DAMTC_UNROLLED_RANK
run default
