#!/bin/bash
mkdir -p gpurun_out
T=${1:-r3e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
./tools/lat_probe > gpurun_out/lat_probe_$T.json 2>&1; cat gpurun_out/lat_probe_$T.json
TS_SHAPES=3,4,6,7,8,13,14,16,17,12 timeout 600 python scripts/tree_shapes.py 10000,100000 > gpurun_out/tree_shapes_$T.jsonl 2>&1; echo shapes rc=$?; cat gpurun_out/tree_shapes_$T.jsonl
