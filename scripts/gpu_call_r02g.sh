#!/bin/bash
# TMA-staged 7-point march: GPU suite, then same-box A/B against the cp.async staging (PC_SMARCH_NO_TMA)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02g_tests.log | head -20
for rep in 1 2; do
  for v in tma cpasync; do
    if [ $v = cpasync ]; then export PC_SMARCH_NO_TMA=1; else unset PC_SMARCH_NO_TMA; fi
    for cfg in c2 c5v c1; do
      st=3; [ $cfg = c5v ] && st=1
      timeout 900 python bench.py --config $cfg --steps $st --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02g_${v}_${cfg}_$rep.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/r02g_${v}_${cfg}_$rep.json').read().strip().splitlines()[-1])
print('$v $cfg rep $rep', '%.4e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))
for r in d['roofline']['all_hot_loops']: print('     ', r['kernel'], '%.1f ms %d launches %.0f GB/s' % (r['ms'], r['launches'], r['achieved']))" 2>&1 | tail -4
    done
  done
done
unset PC_SMARCH_NO_TMA
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scalar_march -s 40 -c 3 -o gpurun_out/r02g_c2_full $CMD > gpurun_out/r02g_c2_full.log 2>&1; echo "ncu c2 rc=$?"
