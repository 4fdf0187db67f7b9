#!/bin/bash
# evidence run of the restored final tree (short, ~30 min): GPU suite + smoke, default C5 line, C3 / C2 / C4 lines,
# the C5 launch list and one ncu --set full capture of the fused stage-1+2 launch and of the plain stage launch
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02g}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 500 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 400 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 700 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python - <<PY
import json
for n in ["c5","c3","c2","c4"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(n, "value %.3e e2e %.3e  %s GB/s frac %s clocks %s power %s" % (d["value"], d["e2e"]["value"], r.get("achieved"), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiStageA12 -s 1 -c 1 -o gpurun_out/${TAG}_a12_full $CMD > gpurun_out/${TAG}_a12_full.log 2>&1; echo "ncu a12 rc=$?"
ncu -i gpurun_out/${TAG}_a12_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_a12_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_a12_full.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 22 -c 2 -o gpurun_out/${TAG}_c5_full $CMD > gpurun_out/${TAG}_c5_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${TAG}_c5_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_c5_full.ncu-rep
