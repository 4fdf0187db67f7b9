#!/bin/bash
# end-of-round-2 evidence on the final code (aligned fused stages 1+2): GPU suite + smoke, full-contract bench lines
# (C5 default, C3, C4, C2, C1, C5v), the reference arm, the C5 launch list and one ncu --set full of the fused launch
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/${TAG}_c1.json 2> gpurun_out/${TAG}_c1.err; echo "c1 rc=$?"
timeout 1500 python bench.py --config c5v --steps 1 --warmup 3 > gpurun_out/${TAG}_c5v.json 2> gpurun_out/${TAG}_c5v.err; echo "c5v rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
python - <<PY
import json
for n in ["c5","c3","c4","c2","c1","c5v","ref"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        if n == "ref":
            print(n, "value %.3e ms_per_step %.3e cores %s" % (d["value"], d["ms_per_step"], d["cpu_baseline"]["cores"])); continue
        r = d.get("roofline") or {}
        print(n, "value %.3e e2e %.3e  %s GB/s frac %s clocks %s power %s" % (d["value"], d["e2e"]["value"], r.get("achieved"), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"].get("power_w")))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 22 -c 3 -o gpurun_out/${TAG}_c5_full $CMD > gpurun_out/${TAG}_c5_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${TAG}_c5_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_c5_full.ncu-rep
