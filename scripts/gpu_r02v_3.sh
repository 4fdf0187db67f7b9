#!/bin/bash
# k_vec_march DM 3 (radial rho read per plane): GPU parity, then C5v with and without it (same box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v7}
timeout 900 python -m pytest tests/test_gpu_vmarch.py tests/test_gpu_c5.py tests/test_gpu_fuse12.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
for v in A B; do
  if [ $v = B ]; then export PC_NO_RADIAL_RHO=1; else unset PC_NO_RADIAL_RHO; fi
  timeout 900 python bench.py --config c5v --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c5v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_${v}_c5v.json').read().strip().splitlines()[-1])
print('$v c5v', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'), 'ms', d['ms_per_step'])
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
done
