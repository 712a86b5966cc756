#!/bin/bash
# CRR changes (leaf-slot trick, strip kernel for N > 1152): tests + config-2 bench; full-kernel shape sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2i.log 2>&1 || { echo build failed; tail gpurun_out/build_r2i.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -k "crr or config2 or tree or european" > gpurun_out/pytest_r2i.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_r2i.log | tail -12
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_r2i.log 2>&1; echo bench2 rc=$?; tail -c 1500 gpurun_out/bench_c2_r2i.log
for v in "-DAMTC_F_WARPS=16 -DAMTC_F_C=4 -DAMTC_F_B=6" "-DAMTC_F_WARPS=16 -DAMTC_F_C=5 -DAMTC_F_B=8" "-DAMTC_F_WARPS=14 -DAMTC_F_C=6 -DAMTC_F_B=8" "-DAMTC_F_WARPS=20 -DAMTC_F_C=4 -DAMTC_F_B=6"; do
  AMTC_NVCC_EXTRA="$v" AB_FORCE=1 AB_MODES=1 AB_SETS=all timeout 600 python scripts/full_ab.py 2>&1 | grep -v "^ *$" | cut -c1-420
done > gpurun_out/full_sweep_r2i.log
cat gpurun_out/full_sweep_r2i.log
