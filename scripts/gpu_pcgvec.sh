# 128-bit PCG update kernels: parity + C4 bench + launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -k "pcg or be or line or c4 or kat or 128bit" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
B="python bench.py --no-cpu-baseline --no-e2e --config c4 --steps 1 --warmup 3"
timeout 900 $B > gpurun_out/pcgvec.json 2> gpurun_out/pcgvec.err; echo "rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/pcgvec.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'), [o['stages_or_iters'] for o in d['config']['operators']])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file gpurun_out/pcgvec_l.csv $B --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_launches.py gpurun_out/pcgvec_l.csv 2>/dev/null | head -8
