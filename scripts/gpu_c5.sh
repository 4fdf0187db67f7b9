cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.used,memory.total --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --config c5 --n 96,96,192 --steps 1 --warmup 1 --cpu-sample-s 5 > gpurun_out/c5s_bench.json 2> gpurun_out/c5s_bench.err; echo "c5 small rc=$?"; tail -5 gpurun_out/c5s_bench.err; cat gpurun_out/c5s_bench.json
timeout 1500 python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err & BP=$!
for i in $(seq 1 150); do sleep 10; if ! kill -0 $BP 2>/dev/null; then break; fi; nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/c5_mem.log; done
wait $BP; echo "c5 full rc=$?"; tail -5 gpurun_out/c5_bench.err; cat gpurun_out/c5_bench.json; tail -3 gpurun_out/c5_mem.log
