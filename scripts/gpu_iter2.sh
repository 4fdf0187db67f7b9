cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s1_bench_$c.json 2> gpurun_out/s1_bench_$c.err
  echo "== $c rc=$?"; tail -3 gpurun_out/s1_bench_$c.err; cut -c1-400 gpurun_out/s1_bench_$c.json
done
timeout 600 python bench.py --config c5 --n 96,96,192 --steps 1 --warmup 1 --cpu-sample-s 5 > gpurun_out/s1_c5s.json 2> gpurun_out/s1_c5s.err; echo "c5s rc=$?"; tail -3 gpurun_out/s1_c5s.err; cat gpurun_out/s1_c5s.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scalar_march -s 12 -c 1 -o gpurun_out/s1_c2_full python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/s1_ncu.log 2>&1; echo "ncu rc=$?"
