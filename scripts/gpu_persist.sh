cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -12
for c in c1 c2; do
for P in 0 1; do
  if [ $P = 1 ]; then export PC_NO_PERSIST=1; else unset PC_NO_PERSIST; fi
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_$c$P.json 2>gpurun_out/p_$c$P.err
  python -c "import json; d=json.loads(open('gpurun_out/p_$c$P.json').read().strip().splitlines()[-1]); print('$c no_persist=$P', d['value'], d['ms_per_step'], d['config']['operators'])" || tail -3 gpurun_out/p_$c$P.err
done
done
