#!/bin/bash
# vector-march r-chunk wave model: C2 (model R = 15) and C5v (model R = 64) against the old fixed R (16 / 32), same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v9}
timeout 900 python -m pytest tests/test_gpu_vmarch.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.log
line() {
  python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$2', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'), 'ms', round(d['ms_per_step'],1))
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
}
for rep in 1 2; do
  for v in model 16; do
    if [ $v = model ]; then unset PC_SMARCH_R; else export PC_SMARCH_R=$v; fi
    timeout 600 python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c2_$rep.json 2>/dev/null
    line gpurun_out/${TAG}_${v}_c2_$rep.json "R=$v c2 rep $rep"
  done
done
for v in model 32; do
  if [ $v = model ]; then unset PC_SMARCH_R; else export PC_SMARCH_R=$v; fi
  timeout 900 python bench.py --config c5v --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c5v.json 2>/dev/null
  line gpurun_out/${TAG}_${v}_c5v.json "R=$v c5v"
done
