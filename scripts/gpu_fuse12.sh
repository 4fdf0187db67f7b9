# fused stage 1+2 (7-point march): parity, C2 bench (fused vs PC_NO_FUSE12), launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_kat_edges.py tests/test_gpu_aligned_visc.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
B="python bench.py --no-cpu-baseline --no-e2e --config c2 --steps 3 --warmup 3"
for V in fused split; do
  if [ $V = split ]; then export PC_NO_FUSE12=1; fi
  timeout 600 $B > gpurun_out/f12_$V.json 2> gpurun_out/f12_$V.err; echo "$V rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/f12_$V.json').read().strip().splitlines()[-1])
print('$V', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'))
for r in d['roofline']['all_hot_loops']: print('   ', r)"
done
unset PC_NO_FUSE12
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/f12_launches.csv $B --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
for q in 1 2; do timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f12_c1_$q.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/f12_c1_$q.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
