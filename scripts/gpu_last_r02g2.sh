#!/bin/bash
# ncu --set full of the plain C5 stage launch (EpiStage) on the final code
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pc::EpiStage," -s 20 -c 1 -o gpurun_out/r02g_st_full $CMD > gpurun_out/r02g_st_full.log 2>&1; echo "ncu stage rc=$?"
ncu -i gpurun_out/r02g_st_full.ncu-rep --page raw --csv > gpurun_out/r02g_st_raw.csv 2>/dev/null
rm -f gpurun_out/r02g_st_full.ncu-rep
