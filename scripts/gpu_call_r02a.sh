cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -m gpu tests/test_gpu_acceptance.py tests/test_gpu_ptl_modes.py 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
CASES="c3 c2 c5r" bash scripts/gpu_parity.sh
