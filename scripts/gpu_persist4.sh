# C1 persistent loop: barrier words on their own lines + poll backoff; 6 processes (bimodality check)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_c1.py tests/test_gpu_kat_edges.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
B="python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for q in 1 2 3 4 5 6; do
  timeout 300 $B > gpurun_out/p4.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/p4.json').read().strip().splitlines()[-1]); print('%.3e' % d['value'], '%.2f ms' % d['ms_per_step'])"
done
