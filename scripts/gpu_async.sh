# asynchronous state uploads / downloads in split_advance: GPU suite + C5/C3 full-contract lines (e2e)
cd $GRAFT_REPO_ROOT
TAG=${1:-as}
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
python - <<PY
import json
for n in ["c5","c3"]:
    d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
    print(n, "value %.3e e2e %.3e (%.0f ms vs %.0f ms)  frac %.3f" % (d["value"], d["e2e"]["value"], d["e2e"]["ms_per_step"], d["ms_per_step"], d["roofline"]["frac"]))
PY
