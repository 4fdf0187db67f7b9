cd $GRAFT_REPO_ROOT
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 300 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err; cat gpurun_out/bench_c1.json
