# C1 per-call step times (3 processes each): persistent loop with cached record buffers, spin barrier
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_c1.py tests/test_gpu_kat_edges.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for q in 1 2 3; do PYTHONPATH=. timeout 300 python scripts/c1_probe.py 2>&1 | tail -1; done
for q in 1 2; do PC_PERSIST_SLEEP=1 PYTHONPATH=. timeout 300 python scripts/c1_probe.py 2>&1 | tail -1; done
for q in 1 2 3; do timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p5.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/p5.json').read().strip().splitlines()[-1]); print('bench %.3e' % d['value'], '%.2f ms' % d['ms_per_step'], d['roofline']['kernel_ms_share'])"; done
