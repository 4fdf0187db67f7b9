#!/bin/bash
# C4 full-size cycle 5 parity (oracle in the background on 14 cores) + the deferred-flush GPU suite and C4 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
python scripts/full_parity.py gpu c4 --from-cycle 4 --max-cycles 1 --out /tmp/full_parity > gpurun_out/full_parity_c4_cycle5.log 2>&1
echo "gpu leg rc=$?"; tail -1 gpurun_out/full_parity_c4_cycle5.log
(timeout 3000 python scripts/full_parity.py oracle c4 --ranks 14 --out /tmp/full_parity --json gpurun_out/full_parity_c4_cycle5.json >> gpurun_out/full_parity_c4_cycle5.log 2>&1; echo "oracle rc=$?" >> gpurun_out/full_parity_c4_cycle5.log) &
OPID=$!
bash scripts/gpu_call_r02m.sh
wait $OPID
tail -3 gpurun_out/full_parity_c4_cycle5.log
