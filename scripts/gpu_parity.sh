#!/bin/bash
# whole-step parity at BASELINE sizes: scripts/full_parity.py per case
# (GPU leg, then the slab oracle on every host core); summaries ->
# gpurun_out/full_parity_<case>.json, logs -> gpurun_out/full_parity_<case>.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
for c in ${CASES:-c3 c2 c5r}; do
  echo "== $c"
  timeout ${PT:-1800} python scripts/full_parity.py both $c --out /tmp/full_parity > gpurun_out/full_parity_$c.log 2>&1
  echo "rc=$?"; tail -4 gpurun_out/full_parity_$c.log
  rm -f /tmp/full_parity/${c}_*.npy
done
