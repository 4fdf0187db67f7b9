# usage: bash scripts/gpu_iter.sh <tag> [configs...]   (runs on the GPU box)
cd $GRAFT_REPO_ROOT
TAG=$1; shift
CFGS=${@:-c3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "== $c rc=$?"; tail -2 gpurun_out/${TAG}_bench_$c.err; cat gpurun_out/${TAG}_bench_$c.json | cut -c1-300
done
if [ -n "$NCU_KERNEL" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$NCU_KERNEL -s ${NCU_SKIP:-5} -c 1 -o gpurun_out/${TAG}_full python bench.py --config ${NCU_CFG:-c3} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
fi
