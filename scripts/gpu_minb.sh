# experiment: smarch launch bounds (3 vs 2 blocks/SM) on C2 (vector viscosity)
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --config c2 --steps 3 --warmup 3"
for V in 3 2; do
  PC_NVCC_EXTRA=-DSMARCH_MINB=$V python -m paper_2403_01004_b200.build --force > /dev/null 2>&1 || echo "build $V failed"
  timeout 600 python -m pytest tests -m gpu -k "visc or vector" -x -q 2>&1 | tail -1
  timeout 600 $B > gpurun_out/minb$V.json 2> gpurun_out/minb$V.err; echo "rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/minb$V.json').read().strip().splitlines()[-1])
print('minb=$V', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'))"
done
