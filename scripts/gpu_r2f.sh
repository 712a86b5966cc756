#!/bin/bash
# the new full solver: build, quick parity tests, A/B vs the strip kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2f.log 2>&1 || { echo build failed; tail gpurun_out/build_r2f.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf --timeout 600 -k "random_small or config1 or edge or warp_path or sawtooth or capacity or fig9 or hedge or european or call_sellers" > gpurun_out/pytest_r2f.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_r2f.log | tail -8
timeout 900 python scripts/full_ab.py > gpurun_out/full_ab_r2f.log 2>&1; echo ab rc=$?; cut -c1-600 gpurun_out/full_ab_r2f.log
