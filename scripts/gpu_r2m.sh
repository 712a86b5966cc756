#!/bin/bash
# race/determinism tests (compute-sanitizer is closed on this pool) + source-level profile of the light kernel (puts)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2m.log 2>&1 || { echo build failed; tail gpurun_out/build_r2m.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_races.py -q -rf --timeout 1100 > gpurun_out/pytest_races_r2m.log 2>&1; echo races rc=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_races_r2m.log | tail -15
timeout 300 python scripts/prof_tc.py 0 1184 1500 > gpurun_out/puts_r2m.log 2>&1; echo run rc=$?; cut -c1-300 gpurun_out/puts_r2m.log
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --section LaunchStats \
   --section Occupancy --section SpeedOfLight --section ComputeWorkloadAnalysis \
   --clock-control none --import-source on -k regex:light_kernel -s 1 -c 1 \
   -o gpurun_out/r2m_light_puts python scripts/prof_tc.py 0 1184 1500 > gpurun_out/ncu_r2m.log 2>&1; echo ncu rc=$?
