mkdir -p gpurun_out
for v in "-DAMTC_TOL_X=1e-13" "-DAMTC_TOL_X=1e-12"; do
  AMTC_NVCC_EXTRA="$v" python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
  tag=$(echo $v | tr -d ' =-')
  AMTC_NVCC_EXTRA="$v" timeout 600 python scripts/bad_sweep.py 2>&1 | head -6
  PH_OUT=gpurun_out/parity_$tag.json timeout 600 python scripts/parity_hist.py > /dev/null 2>&1; echo "$v parity rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/parity_$tag.json'))
for p in ('ask','bid'):
    x=d['config4'][p]; print('$v', p, 'pass', x['pass'], 'floor', x['floor_used'], 'max_units', x['max_err_in_N_eps_S0'], x['abs_err_hist_N_eps_S0'])"
done
python -c "from paper_1110_2477_b200 import build; build.build(force=True)" > /dev/null 2>&1
