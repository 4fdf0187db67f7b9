cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
python scripts/full_parity.py both c4 --out /tmp/full_parity > gpurun_out/full_parity_c4.log 2>&1
echo "rc=$?"; tail -4 gpurun_out/full_parity_c4.log
