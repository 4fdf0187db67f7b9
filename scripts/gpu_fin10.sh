# final evidence with the three-issuer TMA march: GPU suite + smoke, default bench (C5), C3, C4, launch list + ncu of C5 stage
cd $GRAFT_REPO_ROOT
TAG=${1:-fin10}
bash scripts/gpu_full.sh
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python - <<PY
import json
for n in ["c5","c3","c4"]:
    d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
    r=d["roofline"]
    print(n, "value %.3e e2e %.3e  %.0f GB/s frac %.3f clocks %s %s cpu %.2e" % (d["value"], d["e2e"]["value"], r["achieved"], r["frac"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w"), d["cpu_baseline"]["value"]))
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/${TAG}_c5_full $CMD > gpurun_out/${TAG}_c5_full.log 2>&1; echo "ncu full rc=$?"
