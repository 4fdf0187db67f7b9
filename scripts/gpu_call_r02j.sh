#!/bin/bash
# fused p-update + matvec (EpiMatvecP): GPU suite, C4 A/B vs the separate p-update (PC_PCG_NO_FUSEP),
# C4 full-size parity (3 cycles) with the oracle in the background, ncu of the fused iteration kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02j_tests.log 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed|^E  " gpurun_out/r02j_tests.log | head -20
for rep in 1 2; do
  for v in fused sep; do
    if [ $v = sep ]; then export PC_PCG_NO_FUSEP=1; else unset PC_PCG_NO_FUSEP; fi
    timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02j_${v}_c4_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r02j_${v}_c4_$rep.json').read().strip().splitlines()[-1])
print('$v c4 rep $rep', '%.4e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['roofline']['kernel'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'), d['config']['operators'])"
  done
done
unset PC_PCG_NO_FUSEP
python scripts/full_parity.py gpu c4 --max-cycles 3 --out /tmp/full_parity > gpurun_out/full_parity_c4f.log 2>&1; echo "c4 gpu leg rc=$?"
(python scripts/full_parity.py oracle c4 --ranks 14 --out /tmp/full_parity --json gpurun_out/full_parity_c4f.json >> gpurun_out/full_parity_c4f.log 2>&1; echo "oracle rc=$?" >> gpurun_out/full_parity_c4f.log) &
OPID=$!
CMD="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update1v|k_aligned_tma" -s 40 -c 2 -o gpurun_out/r02j_c4_full $CMD > gpurun_out/r02j_c4_full.log 2>&1; echo "ncu c4 rc=$?"
wait $OPID
tail -3 gpurun_out/full_parity_c4f.log
