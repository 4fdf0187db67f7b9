# full-contract bench lines (e2e + cpu_baseline) + launch list of the default config
cd $GRAFT_REPO_ROOT
TAG=${1:-fin}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python bench.py > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"; tail -2 gpurun_out/${TAG}_c5.err
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python - <<PY
import json
for n in ["c5","c3","c4"]:
    try:
        d=json.loads(open("gpurun_out/${TAG}_%s.json"%n).read().strip().splitlines()[-1])
        print(n, "value %.3e e2e %.3e  %.0f GB/s frac %.3f clocks %s cpu %s" % (d["value"], d["e2e"]["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d.get("cpu_baseline",{}).get("value")))
    except Exception as e: print(n, "ERR", e)
PY
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_c5_launches.csv $CMD > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "ncu rc=$?"
