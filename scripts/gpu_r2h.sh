#!/bin/bash
# round 2 re-entry: build, GPU tests (minus the config-4 full batch until its oracle file is complete), smoke,
# full-solver A/B on config-4 subsets + whole batch, bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2h.log 2>&1 || { echo build failed; tail gpurun_out/build_r2h.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 -k "not config4_every_option" > gpurun_out/pytest_r2h.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_r2h.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2h.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_r2h.log
timeout 900 python scripts/full_ab.py > gpurun_out/full_ab_r2h.log 2>&1; echo ab rc=$?; cut -c1-700 gpurun_out/full_ab_r2h.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2h.log 2>&1; echo bench rc=$?; tail -c 3500 gpurun_out/bench_r2h.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2h.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r2h.log 2>&1; echo ncu rc=$?
