#!/bin/bash
# vector 7-point march baseline: C2 bench lines + ncu --set full (source) of the
# fused stage-1+2 launch and the F+argmax launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
for rep in 1 2; do
  timeout 600 python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb_c2_$rep.json 2> gpurun_out/vb_c2_$rep.err; echo "c2 rc=$?"; tail -1 gpurun_out/vb_c2_$rep.json
done
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"SEpiStage12" -s 5 -c 1 -o gpurun_out/vb_f12 $CMD > gpurun_out/vb_f12_ncu.log 2>&1; echo "ncu f12 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_scalar_march<3.*SEpiArgmax" -s 5 -c 1 -o gpurun_out/vb_am $CMD > gpurun_out/vb_am_ncu.log 2>&1; echo "ncu am rc=$?"
for f in vb_f12 vb_am; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/${f}_src.csv 2>/dev/null
done
ls -la gpurun_out
