cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
for R in 1 0; do
  if [ $R = 1 ]; then unset PC_NO_RADIAL_RHO; else export PC_NO_RADIAL_RHO=1; fi
  timeout 1800 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rad$R.json 2> gpurun_out/rad$R.err
  python -c "import json; d=json.loads(open('gpurun_out/rad$R.json').read().strip().splitlines()[-1]); print('radial=$R', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
done
