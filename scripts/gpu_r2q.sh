python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -q -x -k "split or 5b" 2>&1 | tail -2
for v in "-DAMTC_L2_PUB=1" "-DAMTC_L2_PUB=2" "-DAMTC_L2_PUB=4" "-DAMTC_L2_PUB=8"; do
  AMTC_NVCC_EXTRA="$v" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "$v"; timeout 300 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | grep -o "\"config5b[^}]*}"
done
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
