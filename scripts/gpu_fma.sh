# experiment: what -fmad=false (bitwise parity with the numpy oracle) costs at the power cap
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
for V in nofma fma; do
  if [ $V = fma ]; then PC_FMAD=1 python -m paper_2403_01004_b200.build --force > /dev/null 2>&1 || echo "build failed"; fi
  for C in c3 c5; do
    timeout 900 $B --config $C > gpurun_out/fma_${V}_$C.json 2> gpurun_out/fma_${V}_$C.err; echo "$V $C rc=$?"
    python -c "
import json;d=json.loads(open('gpurun_out/fma_${V}_$C.json').read().strip().splitlines()[-1])
print('$V $C', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'), [o['stages_or_iters'] for o in d['config']['operators']])"
  done
done
