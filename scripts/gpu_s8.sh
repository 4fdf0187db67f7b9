cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 900 $B --config c4 --steps 1 --warmup 1 > gpurun_out/s8_c4.json 2> gpurun_out/s8_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/s8_c4.err
python - <<PY
import json
for n in ["c4"]:
    d=json.loads(open("gpurun_out/s8_%s.json"%n).read().strip().splitlines()[-1])
    print(n, "value %.3e  ms/step %.1f  %s %.0f GB/s frac %.3f  clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]), d["config"]["operators"])
PY
CMD="$B --config c4 --steps 1 --warmup 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/s8_c4_launches.csv $CMD > gpurun_out/s8_c4_ncu.log 2>&1; echo "ncu rc=$?"
