#!/bin/bash
# session 6 final validation: full GPU suite, smoke, parity histogram, benches of every config, launch list,
# per-kernel counters of one config-4 step, and a source-level capture of the strip kernel on a small saturated case
mkdir -p gpurun_out
T=${1:-s6e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$T.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$T.log
PH_OUT=gpurun_out/r02_parity_error_hist.json timeout 600 python scripts/parity_hist.py > gpurun_out/parity_$T.log 2>&1; echo parity rc=$?; tail -c 600 gpurun_out/parity_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>gpurun_out/bench_$T.err; echo bench rc=$?; tail -c 1500 gpurun_out/bench_$T.log
for c in 2 5 3 1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_c${c}_$T.log 2>&1; echo bench$c rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu-launches rc=$?
timeout 1500 ncu --clock-control none -k regex:"strip_kernel|light_kernel" -s 2 -c 2 \
   --section LaunchStats --section Occupancy \
   --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
   -o gpurun_out/${T}_step -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$T.log 2>&1; echo ncu-step rc=$?
tail -3 gpurun_out/ncu_step_$T.log
# source-level counters and stall samples: 2,960 calls at N = 400 (one item per warp, saturated CTAs; SASS patching
# makes the kernel many times slower, so the case is small)
AMTC_SPLIT=0 timeout 900 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none \
   -k regex:strip_kernel -c 2 -o gpurun_out/${T}_calls_src -f python scripts/prof_tc.py 1 2960 400 > gpurun_out/ncu_src_$T.log 2>&1; echo ncu-src rc=$?
tail -3 gpurun_out/ncu_src_$T.log
ls -la gpurun_out/*.ncu-rep
