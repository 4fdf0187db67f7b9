cd $GRAFT_REPO_ROOT
PROBE_TIMING=1 PC_GAP_PROFILE=1 PYTHONPATH=. timeout 300 python scripts/step_probe.py c2 2 2>&1 | tail -6
PROBE_TIMING=1 PYTHONPATH=. timeout 300 python scripts/step_probe.py c2 2 2>&1 | tail -4
