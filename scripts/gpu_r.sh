cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -8
for R in 32 default; do
  if [ $R = default ]; then unset PC_MARCH_R; else export PC_MARCH_R=$R; fi
  timeout 1200 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r_c5_$R.json 2>/dev/null
  timeout 1200 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r_c4_$R.json 2>/dev/null
done
unset PC_MARCH_R
python - <<PY
import json
for c in ["c5","c4"]:
    for R in ["32","default"]:
        d=json.loads(open("gpurun_out/r_%s_%s.json"%(c,R)).read().strip().splitlines()[-1])
        print(c, R, "value %.4e  %.0f GB/s frac %.3f clocks %s ms/step %.0f" % (d["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["ms_per_step"]))
PY
