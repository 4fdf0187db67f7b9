cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
for i in 1 2 3; do
  timeout 1800 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/var$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/var$i.json').read().strip().splitlines()[-1]); print('run $i', '%.4e' % d['value'], '%.0f ms' % d['ms_per_step'], '%.0f GB/s' % d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
done
