# per-cycle PTL read: polling vs blocking stream sync (C2, C3), probe + bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -k "cycle or ptl or c1 or fuse" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for V in "PC_X=0" "PC_SYNC_BLOCKING=1"; do
  env $V PYTHONPATH=. timeout 300 python scripts/step_probe.py c2 8 2>&1 | tail -1
  env $V timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sy.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/sy.json').read().strip().splitlines()[-1]); print('[$V] bench c2 %.3e' % d['value'], '%.2f ms' % d['ms_per_step'])"
done
