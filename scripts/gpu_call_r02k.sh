#!/bin/bash
# one reciprocal of rho per node in the 7-point operator: GPU suite, same-box A/B on C5v (ab_prev.so = before)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02k_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02k_tests.log | head -10
for rep in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export PC_LIB_PATH=ab_prev.so; else unset PC_LIB_PATH; fi
    timeout 900 python bench.py --config c5v --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02k_${v}_c5v_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r02k_${v}_c5v_$rep.json').read().strip().splitlines()[-1])
print('$v c5v rep $rep', '%.4e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))
for r in d['roofline']['all_hot_loops']: print('     ', r['kernel'], '%.1f ms %d launches %.0f GB/s' % (r['ms'], r['launches'], r['achieved']))"
  done
done
