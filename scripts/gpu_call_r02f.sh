#!/bin/bash
# folded row records: GPU suite, bench lines, C5 launch list + one full ncu capture of the C5 stage
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/${TAG}_tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="--no-e2e --no-cpu-baseline"
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 $B > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c3 --steps 4 --warmup 3 $B > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 $B > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python - <<PY
import json
for n in ["c5","c3","c4"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        print(n, "value %.3e ms %.1f %.0f GB/s frac %.3f clocks %s power %s" % (d["value"], d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/${TAG}_c5_full $CMD > gpurun_out/${TAG}_c5_full.log 2>&1; echo "ncu full rc=$?"
