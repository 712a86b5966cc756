for v in "" "-DAMTC_DIAG_NO_CFENCE" "-DAMTC_DIAG_NO_PFENCE" "-DAMTC_DIAG_NO_CFENCE -DAMTC_DIAG_NO_PFENCE" "-DAMTC_L2_WARPS=4 -DAMTC_L2_MINB=4"; do
  AMTC_NVCC_EXTRA="$v" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "$v"; timeout 300 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | grep -o "\"config5b[^}]*}" | cut -c1-80
  AMTC_SPLIT=1 timeout 300 python scripts/prof_tc.py 0 8 1500 | cut -c1-200
done
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
