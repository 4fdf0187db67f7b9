# one kernel iteration: GPU parity, C3 bench, one full ncu capture of the fused stage
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B --config c3 --steps 6 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"; tail -2 gpurun_out/${TAG}_c3.err
python - <<PY
import json
d=json.loads(open("gpurun_out/${TAG}_c3.json").read().strip().splitlines()[-1])
print("C3 value %.3e  stage %.0f GB/s frac %.3f  clocks %s" % (d["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]))
PY
CMD="$B --config c3 --steps 1 --warmup 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 12 -c 1 -o gpurun_out/${TAG}_c3_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
