cd $GRAFT_REPO_ROOT
TAG=${1:-c5q}
timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err; echo "c5 rc=$?"; tail -2 gpurun_out/${TAG}.err
python - <<PY
import json
d=json.loads(open("gpurun_out/${TAG}.json").read().strip().splitlines()[-1])
print("C5 value %.3e  ms/step %.0f stage %.0f GB/s frac %.3f  clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]))
PY
