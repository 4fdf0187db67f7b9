cd $GRAFT_REPO_ROOT
for pc in line-r jacobi; do
timeout 1500 python bench.py --config c4 --pc $pc --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c4_$pc.json 2> gpurun_out/c4_$pc.err; echo "$pc rc=$?"; tail -2 gpurun_out/c4_$pc.err
python - <<PY
import json
d=json.loads(open("gpurun_out/c4_$pc.json").read().strip().splitlines()[-1])
print("$pc", "value %.3e ms/step %.1f %s %.0f GB/s frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["achieved"], d["roofline"]["frac"]), d["config"]["operators"], d["config"]["scheme"])
PY
done
CMD="python bench.py --config c4 --pc line-r --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/c4line_launches.csv $CMD > gpurun_out/c4line_ncu.log 2>&1; echo "ncu rc=$?"
