#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02e_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02e_tests.log | head -20
bash scripts/gpu_iter_r02.sh r02e_it 2>&1 | grep -v "^tests rc\|passed\|smoke" | tail -30
CFGS="c3 c4" bash scripts/gpu_tts.sh 2>&1 | tail -16
