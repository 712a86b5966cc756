#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1110_2477_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "light or call_sellers or random_small or config1 or edge" > gpurun_out/pytest_r2c.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_r2c.log
timeout 600 python scripts/light_ab.py > gpurun_out/light_ab_r2c.log 2>&1; echo ab rc=$?; cat gpurun_out/light_ab_r2c.log | cut -c1-400
