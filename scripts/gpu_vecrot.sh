# theta-face rotations with the exact zeros of M skipped (7-point vector march): parity + C2
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -k "visc or vector or fuse or c5 or slab or nccl or kat" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -6
for q in 1 2; do timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vr.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/vr.json').read().strip().splitlines()[-1]); print('c2 %.3e' % d['value'], '%.2f ms' % d['ms_per_step'])"; done
PROBE_TIMING=1 PYTHONPATH=. timeout 300 python scripts/step_probe.py c2 2 2>&1 | tail -4
