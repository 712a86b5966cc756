#!/bin/bash
# full-kernel shape sweep on the GPU box: rebuild with AMTC_FULL_WARPS / AMTC_FULL_CB and time config 4
mkdir -p gpurun_out
CFGS=("${@:-}"); [ -z "$1" ] && CFGS=("20 4" "16 4" "18 4" "16 5")
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  AMTC_NVCC_EXTRA="-DAMTC_FULL_WARPS=$1 -DAMTC_FULL_CB=$2" timeout 600 python -m paper_1110_2477_b200.build --force > /dev/null 2>&1 || { echo "build $1 $2 failed"; continue; }
  timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sweep_w$1_c$2.log 2>&1
  echo "warps=$1 cb=$2 $(python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_w$1_c$2.log').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
