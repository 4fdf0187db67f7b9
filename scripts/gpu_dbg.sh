cd $GRAFT_REPO_ROOT
timeout 300 python -X faulthandler -m pytest tests/test_gpu_aligned_visc.py -x -v -s -k "tma" 2>&1 | tail -40
