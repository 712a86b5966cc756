#!/bin/bash
# strong-scaling slices of the config-4 deal (rank g's share of an n-GPU deal timed alone on this GPU), then
# compute-sanitizer memcheck / racecheck / synccheck on small solver runs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2l.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/slices_r2l.jsonl
for n in 2 4 8; do
  for g in $(seq 0 $((n-1))); do
    timeout 600 python bench.py --slice $g/$n --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/slices_r2l.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/slices_r2l.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    s = d.get("slice", {})
    print(s.get("rank"), "/", s.get("of"), "options", s.get("options"), "ms/step", round(d["ms_per_step"], 1), "cost share", round(s.get("est_cost_share", 0), 4))
PY
bash scripts/gpu_sanitize.sh
