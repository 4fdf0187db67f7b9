# C1: persistent cycle kernel vs host-driven loop (fused stage-1+2 march), 5 runs each (run-to-run spread)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_c1.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
B="python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for q in 1 2 3 4 5; do
  for V in "PC_X=0" "PC_NO_PERSIST=1"; do
    env $V timeout 300 $B > gpurun_out/p3.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/p3.json').read().strip().splitlines()[-1]); print('[$V]', '%.3e' % d['value'], '%.2f ms' % d['ms_per_step'], d['clocks'].get('sm_mhz'))"
  done
done
