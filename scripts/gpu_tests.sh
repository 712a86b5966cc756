#!/bin/bash
# GPU test session: build, the -m gpu suite (optionally filtered), smoke
mkdir -p gpurun_out
TAG=${1:-x}; FILT=${2:-}
python -c "from paper_1110_2477_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
if [ -n "$FILT" ]; then K=(-k "$FILT"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 "${K[@]}" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$TAG.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$TAG.log
