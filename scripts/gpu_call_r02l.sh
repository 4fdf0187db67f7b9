#!/bin/bash
# C4 at full size: the 4th PTL cycle (a long one) through the GPU, the oracle starting from the GPU's state after cycle 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
timeout 3000 python scripts/full_parity.py both c4 --from-cycle 3 --max-cycles 1 --ranks 16 --out /tmp/full_parity \
  --json gpurun_out/full_parity_c4_cycle4.json > gpurun_out/full_parity_c4_cycle4.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/full_parity_c4_cycle4.log
