# final evidence after the async copies: default bench (C5), C4, C2 full-contract lines
cd $GRAFT_REPO_ROOT
TAG=${1:-fin9}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 1200 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
python - <<PY
import json
for n in ["c5","c4","c2"]:
    d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
    r=d["roofline"]
    print(n, "value %.3e e2e %.3e (%.0f vs %.0f ms)  %.0f GB/s frac %.3f traffic %s clocks %s %s" % (d["value"], d["e2e"]["value"], d["e2e"]["ms_per_step"], d["ms_per_step"], r["achieved"], r["frac"], r["traffic"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
PY
