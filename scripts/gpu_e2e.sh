cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kat_edges.py -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 900 python scripts/e2e_profile.py > gpurun_out/e2e_prof.txt 2>&1; echo rc=$?
grep -E "value" gpurun_out/e2e_prof.txt | head -3
sed -n '/ncalls/,+12p' gpurun_out/e2e_prof.txt
