# full GPU suite + C1/C2 full-contract bench lines
cd $GRAFT_REPO_ROOT
TAG=${1:-sm}
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/${TAG}_c1.json 2> gpurun_out/${TAG}_c1.err; echo "c1 rc=$?"
python - <<PY
import json
for n in ["c2","c1"]:
    d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
    print(n, "value %.3e e2e %.3e ms %.2f share %.3f cpu %.2e" % (d["value"], d["e2e"]["value"], d["ms_per_step"], d["roofline"]["kernel_ms_share"], d["cpu_baseline"]["value"]))
PY
