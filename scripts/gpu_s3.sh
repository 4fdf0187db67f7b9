cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.used,memory.total,clocks.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --cpu-sample-s 10 > gpurun_out/s3_c3.json 2> gpurun_out/s3_c3.err; echo "c3 rc=$?"; tail -3 gpurun_out/s3_c3.err; cat gpurun_out/s3_c3.json
timeout 300 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s3_c1.json 2> gpurun_out/s3_c1.err; echo "c1 rc=$?"; tail -3 gpurun_out/s3_c1.err; cut -c1-600 gpurun_out/s3_c1.json
CMD="python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3_c3_launches.csv $CMD > gpurun_out/s3_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_aligned_ -s 30 -c 1 -o gpurun_out/s3_c3_full $CMD > gpurun_out/s3_ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/s3_ncu_full.log
timeout 2400 python bench.py --steps 1 --warmup 3 > gpurun_out/s3_c5.json 2> gpurun_out/s3_c5.err; echo "c5 rc=$?"; tail -5 gpurun_out/s3_c5.err; cat gpurun_out/s3_c5.json
