#!/bin/bash
# source-level profile of the full kernel on 1184 config-4 calls (whole-tree mode)
mkdir -p gpurun_out
T=${1:-r3a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }

timeout 1500 ncu --set full --import-source on --clock-control none -k regex:strip_kernel -s 1 -c 1 \
   -o gpurun_out/${T}_calls python scripts/prof_tc.py 1 1184 1500 > gpurun_out/ncu_$T.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$T.log
