# experiment: k_pcg_update1 variants on C4 (scalar 4 nodes/lane vs 128-bit pairs x1 / x2)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -k "pcg or be or line or c4 or kat" -x -q 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
B="python bench.py --no-cpu-baseline --no-e2e --config c4 --steps 1 --warmup 3"
for V in s 1 2; do
  PC_UPD1=$V timeout 900 $B > gpurun_out/upd_$V.json 2> gpurun_out/upd_$V.err; echo "$V rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/upd_$V.json').read().strip().splitlines()[-1])
print('$V', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'), [o['stages_or_iters'] for o in d['config']['operators']])"
  PC_UPD1=$V timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pcg_update1 -c 20 --csv --log-file gpurun_out/upd_${V}_l.csv $B --steps 1 --warmup 0 > /dev/null 2>&1
  python scripts/ncu_launches.py gpurun_out/upd_${V}_l.csv 2>/dev/null | head -3
done
