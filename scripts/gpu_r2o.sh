#!/bin/bash
# light kernel split mode: parity + race tests, config 5b / 3 / 1 single-tree benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2o.log 2>&1 || { echo build failed; tail gpurun_out/build_r2o.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_tree.py -q -x -rf --timeout 800 -k "split or light or 5b or config1 or races or random_small or edge" > gpurun_out/pytest_r2o.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_r2o.log | tail -12
for c in 5 3 1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c${c}_r2o.log 2>&1; echo bench$c rc=$?; tail -1 gpurun_out/bench_c${c}_r2o.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:60], 'ms/step', round(d['ms_per_step'],2), d.get('config5b'))"; done
