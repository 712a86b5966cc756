#!/bin/bash
# session 6: static snake deal of first items -- parity, bench, 8-GPU slices, calls subset; then source-level
# counters (few passes) of the strip kernel on one config-4 step
mkdir -p gpurun_out
T=${1:-s6c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -m gpu -q -x --timeout 800 > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_$T.log
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_$T.log 2>gpurun_out/bench_$T.err; echo bench rc=$?; tail -c 700 gpurun_out/bench_$T.log
for g in 0 3 7; do timeout 300 python bench.py --slice $g/8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/slices_$T.log 2>>gpurun_out/bench_$T.err; done
timeout 300 python bench.py --slice 0/2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/slices_$T.log 2>>gpurun_out/bench_$T.err
python - <<'PY'
import json
for ln in open("gpurun_out/slices_s6c.log"):
    try: d = json.loads(ln)
    except Exception: continue
    print("slice", d["config"].get("slice"), d["ms_per_step"], d.get("step_ms"))
PY
AMTC_SPLIT=0 timeout 300 python scripts/prof_tc.py 1 2960 1500 > gpurun_out/calls2960_$T.log 2>&1; tail -c 400 gpurun_out/calls2960_$T.log
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --import-source on --clock-control none \
   -k regex:strip_kernel -c 1 -o gpurun_out/${T}_step -f \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$T.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_step_$T.log
ls -la gpurun_out/*.ncu-rep
