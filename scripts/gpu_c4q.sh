cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -k "be_pcg or pcg" 2>&1 | tail -1
CMD="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file gpurun_out/c4q_launches.csv $CMD > gpurun_out/c4q_ncu.log 2>&1; echo "ncu rc=$?"
