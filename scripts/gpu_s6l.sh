#!/bin/bash
# session 6: per-kernel counters (DRAM traffic, FP64 pipe, issue, local traffic) of one config-4 step of the 20 x 3 build
mkdir -p gpurun_out
T=${1:-s6l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 900 ncu --clock-control none -k regex:"strip_kernel|light_kernel" -s 2 -c 2 \
   --section LaunchStats --section Occupancy \
   --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
   -o gpurun_out/${T}_step -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$T.log 2>&1; echo ncu-step rc=$?
ls -la gpurun_out/*.ncu-rep
