# end-of-session check: GPU suite + smoke + the default bench line
cd $GRAFT_REPO_ROOT
bash scripts/gpu_full.sh
timeout 2400 python bench.py > gpurun_out/end_c5.json 2> gpurun_out/end_c5.err; echo "c5 rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/end_c5.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c5 value %.3e e2e %.3e (%.0f vs %.0f ms) frac %.3f clocks %s %s launches %s' % (d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['gpu_launches']))"
