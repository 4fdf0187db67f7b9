#!/bin/bash
# the GPU suite (new files first) + smoke; full log in gpurun_out/gputests.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=15 tests/test_gpu_ptl_modes.py tests/test_gpu_acceptance.py tests/test_gpu_nccl1.py tests/ > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
grep -E "^E  |^FAILED|passed|failed|error" gpurun_out/gputests.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
