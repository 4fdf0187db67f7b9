cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
