#!/bin/bash
# round-2 iteration: GPU suite, bench lines (C5, C3, C2, C5v, C4 short), ncu
# captures of the C2 7-point kernels and the C5 stage
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
mkdir -p gpurun_out
[ -n "$RUN_TESTS" ] && { timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="--no-e2e --no-cpu-baseline"
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 $B > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c3 --steps 4 --warmup 3 $B > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 $B > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c5v --steps 2 --warmup 1 $B > gpurun_out/${TAG}_c5v.json 2> gpurun_out/${TAG}_c5v.err; echo "c5v rc=$?"
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 $B > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python - <<PY
import json
for n in ["c5","c3","c2","c5v","c4"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        print(n, "value %.3e ms %.1f %.0f GB/s frac %.3f clocks %s power %s ops %s" % (d["value"], d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w"), d["config"]["operators"]))
        for r in d["roofline"]["all_hot_loops"]: print("    ", r["kernel"], "%.1f ms %d launches %.0f GB/s" % (r["ms"], r["launches"], r["achieved"]))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scalar_march -s 40 -c 3 -o gpurun_out/${TAG}_c2_full $CMD > gpurun_out/${TAG}_c2_full.log 2>&1; echo "ncu c2 rc=$?"
CMD="python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/${TAG}_c3_full $CMD > gpurun_out/${TAG}_c3_full.log 2>&1; echo "ncu c3 rc=$?"
