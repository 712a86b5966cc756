for v in "" "-DAMTC_TOL_X=1e-12"; do
  AMTC_NVCC_EXTRA="$v" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
  AMTC_NVCC_EXTRA="$v" timeout 600 python scripts/bad_sweep.py
done
