#!/bin/bash
# aligned fused stages 1+2 (EpiStageA12): parity tests, then same-box A/B of C3 / C5 (PC_NO_FUSE12A=1 = two launches), then the full GPU suite
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02y}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuse12a.py tests/test_gpu_aligned_visc.py -q -x > gpurun_out/${TAG}_t1.log 2>&1; echo "fuse12a tests rc=$?"; tail -3 gpurun_out/${TAG}_t1.log
for rep in 1 2; do
for v in on off; do
  if [ $v = off ]; then export PC_NO_FUSE12A=1; else unset PC_NO_FUSE12A; fi
  timeout 600 python bench.py --config c3 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c3_${v}_${rep}.json 2>/dev/null
  timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c5_${v}_${rep}.json 2>/dev/null
done; done
unset PC_NO_FUSE12A
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_c*_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value %.4e ms/step %.1f frac %.3f clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
        for r in d["roofline"].get("all_hot_loops", []): print("   ", r["kernel"], "%.1f ms" % r["ms"], r["launches"], "%.0f GB/s" % r["achieved"])
    except Exception as e: print(f, "ERR", e)
PY
[ -n "$FULL" ] && timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
