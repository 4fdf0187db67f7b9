# experiment: TMA issue spread over 1 / 2 / 3 warps in the TMA march; C5 then C3, interleaved on one box
cd $GRAFT_REPO_ROOT
PC_TMA_SPLIT=3 timeout 900 python -m pytest tests -m gpu -k "aligned or c5 or fullsize or slab or nccl" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for C in c5 c3; do
  for V in 2 3 4 2 3 4; do
    S=1; [ $C = c3 ] && S=6
    PC_TMA_SPLIT=$V timeout 900 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ts.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/ts.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$C [split $V] %.4e' % d['value'], '%.1f GB/s' % r['achieved'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
  done
done
