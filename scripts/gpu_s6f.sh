#!/bin/bash
# session 6: code-size A/B of the heavy block update (instruction-fetch stalls): rebuild on the box per variant
mkdir -p gpurun_out
T=${1:-s6f}
run() {
  name=$1; shift
  AMTC_NVCC_EXTRA="$*" timeout 900 python -m paper_1110_2477_b200.build --force > gpurun_out/build_${T}_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/build_${T}_$name.log; return; }
  timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_$name.log 2>&1
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${T}_$name.log").read().strip().splitlines()[-1])
p = d["parity"]
print("$name", [round(x, 1) for x in d["step_ms"]], "ask", p["ask"]["pass"], p["ask"]["fail"], "bid", p["bid"]["pass"], p["bid"]["fail"], flush=True)
PY
}
if [ "$T" = s6g ]; then
run rolled_lane -DAMTC_ROLLED_SCANS -DAMTC_LANE_MERGED
run rolled_entry -DAMTC_ROLLED_SCANS -DAMTC_ENTRY_KNOWN
run rolled_entry_cross -DAMTC_ROLLED_SCANS -DAMTC_ENTRY_KNOWN -DAMTC_ROLLED_CROSS
run rolled_rank -DAMTC_ROLLED_SCANS -DAMTC_ROLLED_RANK
exit 0
fi
run merged_rolled -DAMTC_SWEEPC_MERGED -DAMTC_ROLLED_SCANS
run all3 -DAMTC_SWEEPC_MERGED -DAMTC_ROLLED_SCANS -DAMTC_LANE_MERGED
run rolled -DAMTC_ROLLED_SCANS
run merged -DAMTC_SWEEPC_MERGED
run base
