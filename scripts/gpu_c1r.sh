cd $GRAFT_REPO_ROOT
for R in 1 2 4 8; do
  PC_SMARCH_R=$R timeout 600 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c1r$R.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c1r$R.json').read().strip().splitlines()[-1]); print('R=$R', d['value'], d['ms_per_step'])"
done
PC_SMARCH_R=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
