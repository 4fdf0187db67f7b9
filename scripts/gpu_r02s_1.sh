#!/bin/bash
# one ncu --set full capture (with source) of the C3 fused Spitzer stage: per-instruction shared-memory conflicts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-s1}
CMD="python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_aligned_tma<pc::EpiStage" -s 20 -c 1 -o gpurun_out/${TAG}_c3 $CMD > gpurun_out/${TAG}_c3.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_c3.ncu-rep --page raw --csv > gpurun_out/${TAG}_c3_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_c3_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_c3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_c3_srcmix.csv 2>/dev/null
ls -la gpurun_out | grep ${TAG}
