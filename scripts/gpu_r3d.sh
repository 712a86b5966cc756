#!/bin/bash
mkdir -p gpurun_out
T=${1:-r3d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
./tools/lat_probe > gpurun_out/lat_probe_$T.json 2>&1; cat gpurun_out/lat_probe_$T.json
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench_$T.log
