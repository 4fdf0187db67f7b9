cd $GRAFT_REPO_ROOT
python -c "import paper_2403_01004_b200._lib as L; print(L.lib().pc_version())" 
timeout 900 python -m pytest tests/test_gpu_c1.py -x -q -m gpu 2>&1 | tail -30
