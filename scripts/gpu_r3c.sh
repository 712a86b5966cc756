#!/bin/bash
mkdir -p gpurun_out
T=${1:-r3c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tree.py -q -x > gpurun_out/pytest_tree_$T.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_tree_$T.log
timeout 600 python scripts/tree_shapes.py > gpurun_out/tree_shapes_$T.jsonl 2>&1; echo shapes rc=$?; cat gpurun_out/tree_shapes_$T.jsonl
AMTC_SPLIT=0 timeout 120 python scripts/prof_tc.py 1 592 700 > gpurun_out/calls700_$T.log 2>&1; echo calls rc=$?; tail -c 400 gpurun_out/calls700_$T.log
AMTC_SPLIT=0 timeout 900 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --import-source on --clock-control none -k regex:strip_kernel -s 1 -c 1 \
   -o gpurun_out/${T}_calls700 python scripts/prof_tc.py 1 592 700 > gpurun_out/ncu_$T.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$T.log
