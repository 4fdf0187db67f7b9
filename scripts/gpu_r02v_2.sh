#!/bin/bash
# k_vec_march: r-chunk length sweep on C2, and a quick C5v line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v5}
for R in 16 8 12 24 32; do
  PC_SMARCH_R=$R timeout 600 python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c2_R$R.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_c2_R$R.json').read().strip().splitlines()[-1])
print('R=$R c2', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'])
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
done
timeout 900 python bench.py --config c5v --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c5v.json 2>gpurun_out/${TAG}_c5v.err; echo "c5v rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_c5v.json').read().strip().splitlines()[-1])
print('c5v', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['ms_per_step'])
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
