#!/bin/bash
AMTC_NVCC_EXTRA="-DAMTC_L2_PROF=1" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 300 python scripts/prof_light_split.py
for v in "" "-DAMTC_L2_WARPS=6"; do
  AMTC_NVCC_EXTRA="$v" AB_FORCE=1 AB_ALL=1 timeout 600 python scripts/light_ab.py 2>&1 | grep '"set"' | grep -v '"mode": 2' | cut -c1-300
done
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
