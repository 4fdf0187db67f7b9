cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
timeout 600 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1d.json 2> gpurun_out/c1d.err; echo "c1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c1d.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'])"
