cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -6
CMD="python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/s5_c5_full $CMD > gpurun_out/s5_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/s5_ncu.log
