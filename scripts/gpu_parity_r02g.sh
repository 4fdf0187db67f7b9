#!/bin/bash
# whole-step parity on the restored final code (aligned stages 1+2 fused): the C5 recipe on 128x128x256, C3 (RKL2, then RKG2) at BASELINE size
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c5r c3 c3g; do
  timeout 600 python scripts/full_parity.py both $c --ranks 16 --json gpurun_out/r02g_full_parity_$c.json > gpurun_out/r02g_parity_$c.log 2>&1
  echo "$c rc=$?"; tail -3 gpurun_out/r02g_parity_$c.log | cut -c1-400
done
