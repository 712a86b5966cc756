#!/bin/bash
# source-level ncu capture of the full solver on the whole config-4 batch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2g.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/run_c4.py 1 > gpurun_out/run_c4_r2g.log 2>&1; echo run rc=$?; cat gpurun_out/run_c4_r2g.log
timeout 2400 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --section LaunchStats \
   --section Occupancy --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis \
   --clock-control none --import-source on -k regex:full_kernel -s 1 -c 1 \
   -o gpurun_out/r2g_full python scripts/run_c4.py 1 > gpurun_out/ncu_r2g.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_r2g.log
