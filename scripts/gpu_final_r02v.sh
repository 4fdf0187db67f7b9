#!/bin/bash
# end-of-round-2 evidence (after the vector march, csrc/vmarch.cuh): GPU suite + smoke, full-contract bench lines (C5 default, C3, C4, C2, C1, C5v),
# the reference arm, the C5 launch list and full ncu captures (C5 stage, C4 PCG kernels)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02v}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
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
        print(n, "value %.3e e2e %.3e  %.0f GB/s frac %.3f clocks %s power %s cpu %.3e" % (d["value"], d["e2e"]["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w"), d["cpu_baseline"]["value"]))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/${TAG}_c5_full $CMD > gpurun_out/${TAG}_c5_full.log 2>&1; echo "ncu full rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update1v|k_pcg_pupdatev|k_aligned_tma" -s 40 -c 3 -o gpurun_out/${TAG}_c4_full $CMD > gpurun_out/${TAG}_c4_full.log 2>&1; echo "ncu c4 rc=$?"
CMD="python bench.py --config c5v --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_vec_march" -s 6 -c 3 -o gpurun_out/${TAG}_c5v_full $CMD > gpurun_out/${TAG}_c5v_full.log 2>&1; echo "ncu c5v rc=$?"
ncu -i gpurun_out/${TAG}_c5v_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5v_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_c5v_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_c5v_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_c5_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_c4_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_c4_raw.csv 2>/dev/null
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv $CMD > /dev/null 2>&1; echo "ncu c2 list rc=$?"
rm -f gpurun_out/${TAG}_c4_full.ncu-rep gpurun_out/${TAG}_c5_full.ncu-rep
