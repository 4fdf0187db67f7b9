#!/bin/bash
# C4 full-size parity (first 3 PTL cycles: 8 + ~100 PCG iterations) with its
# oracle leg on the host cores in the background, while the GPU runs the
# test suite and ncu captures (nothing timing-sensitive in this call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
python scripts/full_parity.py gpu c4 --max-cycles 3 --out /tmp/full_parity > gpurun_out/full_parity_c4.log 2>&1
echo "c4 gpu leg rc=$?"
(python scripts/full_parity.py oracle c4 --ranks 13 --out /tmp/full_parity >> gpurun_out/full_parity_c4.log 2>&1; echo "oracle rc=$?" >> gpurun_out/full_parity_c4.log) &
OPID=$!
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02d_tests.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scalar_march -s 40 -c 3 -o gpurun_out/r02d_c2_full $CMD > gpurun_out/r02d_c2_full.log 2>&1; echo "ncu c2 rc=$?"
CMD="python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_aligned_tma -s 20 -c 1 -o gpurun_out/r02d_c3_full $CMD > gpurun_out/r02d_c3_full.log 2>&1; echo "ncu c3 rc=$?"
wait $OPID
tail -4 gpurun_out/full_parity_c4.log
