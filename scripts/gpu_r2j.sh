#!/bin/bash
# where the full solvers spend their time: amtc_full.cu phase counters (-DAMTC_F_PROF=1) on the whole batch and on
# 3000 calls; then a source-level ncu capture of the default strip kernel on 3000 calls (whole-tree mode)
mkdir -p gpurun_out
AMTC_NVCC_EXTRA="-DAMTC_F_PROF=1" PF_FORCE=1 timeout 900 python -c "
import os,sys; sys.argv=['x']; os.environ['AB']='1'
" ; AMTC_NVCC_EXTRA="-DAMTC_F_PROF=1" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > gpurun_out/build_prof_r2j.log 2>&1 || { echo build failed; exit 1; }
python - > gpurun_out/prof_full_r2j.log 2>&1 <<'PY'
import sys; sys.argv = ["prof_full.py", "all", "calls3000"]
from paper_1110_2477_b200 import api
api.lib(); api.debug_set_full_kernel(1)
exec(open("scripts/prof_full.py").read().replace("build.build(force=os.environ.get(\"PF_FORCE\") == \"1\"); api.lib()", "api.lib()"))
PY
echo prof rc=$?; cut -c1-900 gpurun_out/prof_full_r2j.log
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > gpurun_out/build_r2j.log 2>&1 || { echo build failed; exit 1; }
AMTC_SPLIT=0 timeout 300 python scripts/prof_tc.py 1 3000 1500 > gpurun_out/calls3000_r2j.log 2>&1; echo run rc=$?; cat gpurun_out/calls3000_r2j.log | cut -c1-400
AMTC_SPLIT=0 timeout 2400 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --section LaunchStats \
   --section Occupancy --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis \
   --clock-control none --import-source on -k regex:strip_kernel -s 1 -c 1 \
   -o gpurun_out/r2j_strip_calls3000 python scripts/prof_tc.py 1 3000 1500 > gpurun_out/ncu_r2j.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_r2j.log
