#!/bin/bash
# re-entry check of the restored tree (round 2, last session): GPU suite + smoke + the default bench line (C5), C2 and C3
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
python - <<PY
import json
for n in ["c5","c2","c3"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        print(n, "value %.3e e2e %.3e  %.0f GB/s frac %.3f clocks %s power %s" % (d["value"], d["e2e"]["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
    except Exception as e: print(n, "ERR", e)
PY
