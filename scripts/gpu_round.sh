#!/bin/bash
# one GPU session: tests, heavy/light micro-runs, bench (config 4, 1 step)
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q --timeout 800 > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
timeout 300 python scripts/prof_tc.py 1 1 1500 > gpurun_out/call1_$TAG.log 2>&1; echo call1 rc=$?
timeout 600 python scripts/prof_tc.py 1 1184 1500 > gpurun_out/calls_$TAG.log 2>&1; echo calls rc=$?
timeout 300 python scripts/prof_tc.py 0 1184 1500 > gpurun_out/puts_$TAG.log 2>&1; echo puts rc=$?
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo bench rc=$?
