# experiment: smarch r-chunk length on C2 (2 blocks/SM vector kernels)
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --config c2 --steps 3 --warmup 3"
for R in def 4 16 32; do
  if [ $R = def ]; then unset PC_SMARCH_R; else export PC_SMARCH_R=$R; fi
  timeout 600 $B > gpurun_out/smr$R.json 2> gpurun_out/smr$R.err; echo "rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/smr$R.json').read().strip().splitlines()[-1])
print('R=$R', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['kernel_ms_share'], d['clocks'].get('sm_mhz'))"
done
unset PC_SMARCH_R
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c2l.csv $B --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
