#!/bin/bash
# session 6: full-kernel slot-count A/B with the rolled-scan build (20 warps x 3 / 4 vertex slots)
mkdir -p gpurun_out
bash scripts/warp_sweep.sh "20 3" "20 4" 2>&1 | tee gpurun_out/sweep_s6j.log
for cfg in "20 3" "20 4"; do set -- $cfg; python - <<PY
import json
d = json.loads(open("gpurun_out/sweep_w$1_c$2.log").read().strip().splitlines()[-1])
print("$1x$2", d["step_ms"], d["parity"]["ask"]["fail"], d["parity"]["bid"]["fail"], d["config"].get("retried_items"))
PY
done
