# full GPU suite + smoke, then the full-contract bench lines of every config and the C5 ncu evidence
cd $GRAFT_REPO_ROOT
bash scripts/gpu_full.sh
bash scripts/gpu_final2.sh ${1:-fin6}
