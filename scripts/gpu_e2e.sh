cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
for c in c3 c5; do
  timeout 1800 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err; echo "$c rc=$?"; tail -3 gpurun_out/e2e_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e'])"
done
