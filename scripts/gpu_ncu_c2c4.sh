# one ncu --set full capture each: C2 fused stage-1+2 launch, C4 128-bit x/r-update and p-update
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:SEpiStage12 -s 5 -c 1 -o gpurun_out/c2f12_full python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/c2f12_ncu.log 2>&1; echo "c2 rc=$?"
