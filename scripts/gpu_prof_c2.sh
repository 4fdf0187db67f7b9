cd $GRAFT_REPO_ROOT
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scalar_march" -s 20 -c 2 -o gpurun_out/p2_full $CMD > gpurun_out/p2_ncu.log 2>&1; echo "ncu rc=$?"
