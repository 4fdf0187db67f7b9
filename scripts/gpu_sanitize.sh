#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_cases.py);
# logs -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
echo "== host"; nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread" ; nvidia-smi --query-gpu=name,memory.total --format=csv
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_cases.py ${CASES:-} \
     > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
