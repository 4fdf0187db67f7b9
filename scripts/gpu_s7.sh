cd $GRAFT_REPO_ROOT
for c in c4 c2; do
CMD="python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s7_${c}_launches.csv $CMD > gpurun_out/s7_${c}_ncu.log 2>&1; echo "$c ncu rc=$?"
done
