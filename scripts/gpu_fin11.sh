# final code, default bench line (C5) + C3 on a fresh box
cd $GRAFT_REPO_ROOT
TAG=${1:-fin11}
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"

python - <<PY
import json
for n in ["c5"]:
    d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
    r=d["roofline"]
    print(n, "value %.3e e2e %.3e  %.0f GB/s frac %.3f clocks %s %s" % (d["value"], d["e2e"]["value"], r["achieved"], r["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
PY
