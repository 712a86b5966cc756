#!/bin/bash
# session 6: A/B of the sweep-A change on config 4 + a source-level ncu capture of the strip kernel on 2,960 calls
mkdir -p gpurun_out
T=${1:-s6b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 800 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_$T.log
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.log 2>gpurun_out/bench_$T.err; echo bench rc=$?; tail -c 1500 gpurun_out/bench_$T.log
AMTC_SPLIT=0 timeout 300 python scripts/prof_tc.py 1 2960 1500 > gpurun_out/calls2960_$T.log 2>&1; tail -c 600 gpurun_out/calls2960_$T.log
AMTC_SPLIT=0 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:strip_kernel -c 2 -o gpurun_out/${T}_calls -f \
   python scripts/prof_tc.py 1 2960 1500 > gpurun_out/ncu_calls_$T.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_calls_$T.log
ls -la gpurun_out/*.ncu-rep
