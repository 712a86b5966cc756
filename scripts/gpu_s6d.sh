#!/bin/bash
# session 6: every slice of the 2/4/8-GPU deals with the snake deal, then a full-kernel shape sweep with the
# leaner sweep A (rebuilds on the box; the default shape is rebuilt last)
mkdir -p gpurun_out
T=${1:-s6d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1 || { echo build failed; tail gpurun_out/build_$T.log; exit 1; }
rm -f gpurun_out/slices_$T.jsonl
for n in 8 4 2; do for ((g=0; g<n; g++)); do
  timeout 300 python bench.py --slice $g/$n --steps 2 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/slices_$T.jsonl 2>>gpurun_out/slices_$T.err
done; done
python - <<PY
import json
for ln in open("gpurun_out/slices_$T.jsonl"):
    try: d = json.loads(ln)
    except Exception: continue
    print("slice", d.get("slice"), round(d["ms_per_step"], 1))
PY
bash scripts/warp_sweep.sh "18 4" "16 4" "16 6" "20 4" 2>&1 | tee gpurun_out/sweep_$T.log
