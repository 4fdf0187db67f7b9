cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/c1f.json 2> gpurun_out/c1f.err; echo "c1 rc=$?"; tail -2 gpurun_out/c1f.err
python -c "import json; d=json.loads(open('gpurun_out/c1f.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['achieved'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'])"
