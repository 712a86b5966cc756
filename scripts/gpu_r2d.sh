#!/bin/bash
mkdir -p gpurun_out
for v in "-DAMTC_L2_B=8" "-DAMTC_L2_B=8 -DAMTC_L2_GFALLBACK=0" "-DAMTC_L2_B=10 -DAMTC_L2_GFALLBACK=0 -DAMTC_L2_WARPS=8" "-DAMTC_L2_B=6 -DAMTC_L2_WARPS=12"; do
  AMTC_NVCC_EXTRA="$v" AB_FORCE=1 AB_ALL=1 timeout 600 python scripts/light_ab.py 2>&1 | grep -v "^ *$" | cut -c1-330
done > gpurun_out/light_ab_r2d.log
cat gpurun_out/light_ab_r2d.log
