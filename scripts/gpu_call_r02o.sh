#!/bin/bash
# C4 full-size cycle 6 (the last, ~420 PCG iterations) parity, the oracle on all 16 host cores from the GPU's state after cycle 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
timeout 3400 python scripts/full_parity.py both c4 --from-cycle 5 --max-cycles 1 --ranks 16 --out /tmp/full_parity \
  --json gpurun_out/full_parity_c4_cycle6.json > gpurun_out/full_parity_c4_cycle6.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/full_parity_c4_cycle6.log
