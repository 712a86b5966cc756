#!/bin/bash
# light kernel: cp.async carry prefetch + per-item constants in shared memory; shape variants; puts parity
mkdir -p gpurun_out
for v in "" "-DAMTC_L2_WARPS=6" "-DAMTC_L2_WARPS=6 -DAMTC_L2_MINB=3"; do
  AMTC_NVCC_EXTRA="$v" AB_FORCE=1 AB_ALL=0 timeout 600 python scripts/light_ab.py 2>&1 | grep -v "^ *$" | cut -c1-330
done > gpurun_out/light_ab_r2n.log
cat gpurun_out/light_ab_r2n.log
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf --timeout 600 -k "random_small or config1 or edge or light or call_sellers or european or hedge or fig9" > gpurun_out/pytest_r2n.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_r2n.log | tail -8
