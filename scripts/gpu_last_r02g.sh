#!/bin/bash
# last short call: ncu --set full of the plain C5 stage launch on the final code, the C1 line, the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiStage, 2" -s 20 -c 1 -o gpurun_out/r02g_st_full $CMD > gpurun_out/r02g_st_full.log 2>&1; echo "ncu stage rc=$?"
ncu -i gpurun_out/r02g_st_full.ncu-rep --page raw --csv > gpurun_out/r02g_st_raw.csv 2>/dev/null
rm -f gpurun_out/r02g_st_full.ncu-rep
timeout 120 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r02g_c1.json 2> gpurun_out/r02g_c1.err; echo "c1 rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02g_ref.json 2> gpurun_out/r02g_ref.err; echo "ref rc=$?"
