#!/bin/bash
# deferred per-plane PCG flush (plane_begin): GPU suite + same-box A/B on C4 and C3-BE (ab_prev.so = before)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02m_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02m_tests.log | head -10
for rep in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export PC_LIB_PATH=ab_prev.so; else unset PC_LIB_PATH; fi
    timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02m_${v}_c4_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r02m_${v}_c4_$rep.json').read().strip().splitlines()[-1])
print('$v c4 rep $rep', '%.4e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
  done
done
