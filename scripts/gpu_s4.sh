cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B --config c3 --steps 2 --warmup 3 > gpurun_out/s4_c3.json 2> gpurun_out/s4_c3.err; echo "c3 rc=$?"; tail -2 gpurun_out/s4_c3.err; cut -c1-300 gpurun_out/s4_c3.json; grep -o '"roofline.*' gpurun_out/s4_c3.json | cut -c1-200
timeout 1500 $B --config c5 --steps 1 --warmup 1 > gpurun_out/s4_c5.json 2> gpurun_out/s4_c5.err; echo "c5 rc=$?"; tail -2 gpurun_out/s4_c5.err; cut -c1-300 gpurun_out/s4_c5.json; grep -o '"roofline.*' gpurun_out/s4_c5.json | cut -c1-200
timeout 1800 $B --config c4 --steps 1 --warmup 1 > gpurun_out/s4_c4.json 2> gpurun_out/s4_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/s4_c4.err; cat gpurun_out/s4_c4.json
