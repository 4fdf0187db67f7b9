#!/bin/bash
# 7-point march staging A/B on one box: cp.async (default) vs TMA (PC_SMARCH_TMA=1); + the opt-in parity test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_poison.py tests/test_gpu_fuse12.py tests/test_gpu_c1.py -q -m gpu > gpurun_out/r02h_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02h_tests.log
for rep in 1 2; do
  for v in cpasync tma; do
    if [ $v = tma ]; then export PC_SMARCH_TMA=1; else unset PC_SMARCH_TMA; fi
    for cfg in c2 c5v; do
      st=3; [ $cfg = c5v ] && st=1
      w=2; [ $cfg = c5v ] && w=1
      timeout 900 python bench.py --config $cfg --steps $st --warmup $w --no-e2e --no-cpu-baseline > gpurun_out/r02h_${v}_${cfg}_$rep.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/r02h_${v}_${cfg}_$rep.json').read().strip().splitlines()[-1])
print('$v $cfg rep $rep', '%.4e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))
for r in d['roofline']['all_hot_loops']: print('     ', r['kernel'], '%.1f ms %d launches %.0f GB/s' % (r['ms'], r['launches'], r['achieved']))" 2>&1 | tail -4
    done
  done
done
