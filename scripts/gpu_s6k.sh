#!/bin/bash
# session 6: validation of the 20-warp x 3-slot full kernel: full GPU suite, smoke, config-4 bench, launch list
mkdir -p gpurun_out
T=${1:-s6k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$T.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>gpurun_out/bench_$T.err; echo bench rc=$?; tail -c 400 gpurun_out/bench_$T.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu-launches rc=$?
