#!/bin/bash
# round 2, first GPU session: baseline tests + class timings + light-kernel source profile
mkdir -p gpurun_out
python -c "from paper_1110_2477_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_r2a.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_r2a.log
timeout 600 python scripts/diag_tc.py 1500 256,1024 > gpurun_out/diag_r2a.log 2>&1; echo diag rc=$?
cat gpurun_out/diag_r2a.log | cut -c1-300
timeout 300 python scripts/prof_tc.py 0 1184 1500 > gpurun_out/puts_r2a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:strip_kernel -c 1 \
   -o gpurun_out/r2a_puts python scripts/prof_tc.py 0 1184 1500 > gpurun_out/ncu_r2a.log 2>&1; echo ncu rc=$?
