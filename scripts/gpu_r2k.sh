#!/bin/bash
# round 2 validation: full GPU suite (incl. every config-4 option vs the oracle), smoke, parity histogram, bench,
# launch list, DRAM traffic of the benched solver kernels (one --set full capture of the step's strip kernel)
mkdir -p gpurun_out
T=${1:-r2k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$T.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$T.log
timeout 600 python scripts/parity_hist.py > gpurun_out/parity_$T.log 2>&1; echo parity rc=$?; tail -c 1500 gpurun_out/parity_$T.log
cp profiles/r02_parity_error_hist.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo bench rc=$?; tail -c 4000 gpurun_out/bench_$T.log
for c in 2 5 3 1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_c${c}_$T.log 2>&1; echo bench$c rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu-launches rc=$?
timeout 2400 ncu --set full --clock-control none -k regex:"strip_kernel|light_kernel" -s 2 -c 2 -o gpurun_out/${T}_full_step \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$T.log 2>&1; echo ncu-full rc=$?
tail -3 gpurun_out/ncu_full_$T.log
