cd $GRAFT_REPO_ROOT
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_aligned_march -s 20 -c 1 -o gpurun_out/prof_march $CMD > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/ncu.log
