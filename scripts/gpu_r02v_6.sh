#!/bin/bash
# k_vec_march tile height: 16-row tiles (512 threads, 1 block/SM; PC_VMARCH_TJ=16) vs 8-row tiles, same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v11}
PC_VMARCH_TJ=16 timeout 900 python -m pytest tests/test_gpu_vmarch.py tests/test_gpu_c5.py tests/test_gpu_fuse12.py tests/test_gpu_nccl1.py tests/test_gpu_slab_local.py -x -q > gpurun_out/${TAG}_tests16.log 2>&1; echo "tests TJ=16 rc=$?"; tail -2 gpurun_out/${TAG}_tests16.log
line() {
  python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$2', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'), 'ms', round(d['ms_per_step'],1))
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
}
for rep in 1 2; do
  for v in 16 8; do
    export PC_VMARCH_TJ=$v
    timeout 600 python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c2_$rep.json 2>/dev/null
    line gpurun_out/${TAG}_${v}_c2_$rep.json "TJ=$v c2 rep $rep"
  done
done
for v in 16 8; do
  export PC_VMARCH_TJ=$v
  timeout 900 python bench.py --config c5v --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c5v.json 2>/dev/null
  line gpurun_out/${TAG}_${v}_c5v.json "TJ=$v c5v"
done
