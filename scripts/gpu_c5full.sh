cd $GRAFT_REPO_ROOT
free -g | head -2
timeout 1700 python bench.py > gpurun_out/c5full_bench.json 2> gpurun_out/c5full_bench.err & BP=$!
for i in $(seq 1 170); do sleep 10; if ! kill -0 $BP 2>/dev/null; then break; fi; nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/c5full_mem.log; free -g | sed -n 2p >> gpurun_out/c5full_hostmem.log; done
wait $BP; echo "rc=$?"; tail -5 gpurun_out/c5full_bench.err; cat gpurun_out/c5full_bench.json; sort -n gpurun_out/c5full_mem.log | tail -1
