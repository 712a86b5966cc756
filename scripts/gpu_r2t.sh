#!/bin/bash
# light split mode with opportunistic staging: tests + 5b for publication cadences; light kernel shape on the full batch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -q -x -k "split or 5b or light" 2>&1 | tail -2
for v in "-DAMTC_L2_PUB=1" "-DAMTC_L2_PUB=2" "-DAMTC_L2_PUB=4"; do
  AMTC_NVCC_EXTRA="$v" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "$v"; timeout 300 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | grep -o "\"config5b[^}]*}" | cut -c1-90
  AMTC_SPLIT=1 timeout 300 python scripts/prof_tc.py 0 8 1500 | cut -c1-200
done
for v in "" "-DAMTC_L2_WARPS=6"; do
  AMTC_NVCC_EXTRA="$v" AB_FORCE=1 AB_ALL=1 timeout 600 python scripts/light_ab.py 2>&1 | grep '"set"' | grep -v '"mode": 2' | cut -c1-260
done
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
