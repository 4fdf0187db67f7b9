#!/bin/bash
# whole-step parity on the final code (aligned stages 1+2 fused): C3 (RKL2 and RKG2) at BASELINE size, the C5 recipe on 128x128x256
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c5r c3 c3g; do
  timeout 1500 python scripts/full_parity.py both $c --ranks 16 --json gpurun_out/r02f_full_parity_$c.json > gpurun_out/r02f_parity_$c.log 2>&1
  echo "$c rc=$?"; tail -3 gpurun_out/r02f_parity_$c.log | cut -c1-400
done
# one ncu --set full capture of the fused stage-1+2 launch at C5 size (the second one: u1 written, s >= 3)
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiStageA12 -s 1 -c 1 -o gpurun_out/r02f_a12_full $CMD > gpurun_out/r02f_a12_full.log 2>&1; echo "ncu a12 rc=$?"
ncu -i gpurun_out/r02f_a12_full.ncu-rep --page raw --csv > gpurun_out/r02f_a12_raw.csv 2>/dev/null
rm -f gpurun_out/r02f_a12_full.ncu-rep
