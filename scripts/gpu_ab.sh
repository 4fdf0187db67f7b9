#!/bin/bash
# same-box A/B of two in-tree builds (PC_LIB_PATH): default .so (A) vs ${B:-ab_nofold.so}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BS=${B:-ab_nofold.so}
for rep in 1 2; do
  for v in A B; do
    for cfg in ${CFGS:-c5 c3}; do
      if [ $v = B ]; then export PC_LIB_PATH=$BS; else unset PC_LIB_PATH; fi
      st=2; [ $cfg = c3 ] && st=4
      timeout 900 python bench.py --config $cfg --steps $st --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_${cfg}_$rep.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/ab_${v}_${cfg}_$rep.json').read().strip().splitlines()[-1])
print('$v $cfg rep $rep', '%.4e'%d['value'], 'frac %.4f'%d['roofline']['frac'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
    done
  done
done
