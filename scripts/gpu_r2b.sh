#!/bin/bash
# round 2 session b: source-level profiles of the light kernel (puts) and the full kernel (call buyers)
mkdir -p gpurun_out
python -c "from paper_1110_2477_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/prof_tc.py 0 1184 1500 > gpurun_out/puts_r2b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:strip_kernel -s 3 -c 1 \
   -o gpurun_out/r2b_puts python scripts/prof_tc.py 0 1184 1500 > gpurun_out/ncu_r2b_puts.log 2>&1; echo ncu puts rc=$?
timeout 300 python scripts/prof_tc.py 1 24 1500 > gpurun_out/calls24_r2b.log 2>&1 && \
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --section LaunchStats \
   --section Occupancy --section SpeedOfLight --section MemoryWorkloadAnalysis --clock-control none --import-source on \
   -k regex:strip_kernel -s 2 -c 1 \
   -o gpurun_out/r2b_calls python scripts/prof_tc.py 1 24 1500 > gpurun_out/ncu_r2b_calls.log 2>&1; echo ncu calls rc=$?
cat gpurun_out/puts_r2b.log gpurun_out/calls24_r2b.log | cut -c1-400
