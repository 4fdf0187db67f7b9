cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -k "pcg or be or line or c4 or kat or 128bit" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
timeout 900 python bench.py --no-cpu-baseline --no-e2e --config c4 --steps 1 --warmup 3 > gpurun_out/pv2.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/pv2.json').read().strip().splitlines()[-1]); print('c4 %.3e' % d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
