# persistent cycle kernel with stages 1+2 fused: parity + C1 bench (fused vs previous numbers)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_c1.py tests/test_gpu_kat_edges.py tests/test_gpu_cli.py tests/test_gpu_analysis.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
for q in 1 2; do timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p2_c1_$q.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/p2_c1_$q.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
