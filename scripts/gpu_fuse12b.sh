# fused stage 1+2, ring operands: parity + C2 bench + launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fuse12.py tests/test_gpu_kat_edges.py tests/test_gpu_aligned_visc.py tests/test_gpu_c1.py -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
B="python bench.py --no-cpu-baseline --no-e2e --config c2 --steps 3 --warmup 3"
timeout 600 $B > gpurun_out/f12b.json 2> gpurun_out/f12b.err; echo "rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/f12b.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'))
for r in d['roofline']['all_hot_loops']: print('   ', r)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/f12b_launches.csv $B --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_launches.py gpurun_out/f12b_launches.csv | head -5
