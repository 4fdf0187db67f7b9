cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B --config c3 --steps 6 --warmup 3 > gpurun_out/s6_c3.json 2> gpurun_out/s6_c3.err; echo "c3 rc=$?"
timeout 900 $B --config c4 --steps 1 --warmup 1 > gpurun_out/s6_c4.json 2> gpurun_out/s6_c4.err; echo "c4 rc=$?"
timeout 600 $B --config c2 --steps 2 --warmup 3 > gpurun_out/s6_c2.json 2> gpurun_out/s6_c2.err; echo "c2 rc=$?"
python - <<PY
import json
for n in ["c3","c4","c2"]:
    try:
        d=json.loads(open("gpurun_out/s6_%s.json"%n).read().strip().splitlines()[-1])
        print(n, "value %.3e  ms/step %.1f  %s %.0f GB/s frac %.3f  clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
    except Exception as e: print(n, "ERR", e)
PY
