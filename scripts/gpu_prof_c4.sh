cd $GRAFT_REPO_ROOT
CMD="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/p4_plain.json 2>/dev/null; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aligned_tma|k_pcg_update1|k_pcg_pupdate" -s 40 -c 3 -o gpurun_out/p4_full $CMD > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/p4_ncu.log
