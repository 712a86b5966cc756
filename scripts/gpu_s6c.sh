#!/bin/bash
# session 6: source-level counters (few passes) of the strip kernel on one config-4 step
mkdir -p gpurun_out
T=${1:-s6c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --import-source on --clock-control none \
   -k regex:"strip_kernel<4" -c 1 -o gpurun_out/${T}_step -f \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$T.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_step_$T.log
ls -la gpurun_out/*.ncu-rep
