#!/bin/bash
# heavy-update tweaks (unrolled WV3 stores, ballot prefix sums): parity on heavy paths + config-4 timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -q -rf --timeout 1100 -k "warp_path or sawtooth or config4 or races or capacity or random_small or split" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('config4 ms/step', d['ms_per_step'], d['parity']['ask']['fail'], d['parity']['bid']['fail'], d['roofline']['kernels']['full']['ms'])"
