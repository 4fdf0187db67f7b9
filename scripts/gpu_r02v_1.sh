#!/bin/bash
# k_vec_march: GPU parity (new tests + the vector suites), C2 A/B against k_scalar_march, ncu of the new kernels
cd $GRAFT_REPO_ROOT
TAG=${1:-v1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vmarch.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "vmarch tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
[ -n "$SUITES" ] && timeout 900 python -m pytest $SUITES -x -q > gpurun_out/${TAG}_tests2.log 2>&1; echo "vector suites rc=$?"; tail -3 gpurun_out/${TAG}_tests2.log
for rep in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export PC_NO_VMARCH=1; else unset PC_NO_VMARCH; fi
    timeout 600 python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${v}_c2_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_${v}_c2_$rep.json').read().strip().splitlines()[-1])
print('$v c2 rep $rep', '%.4e'%d['value'], 'MHz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))
for h in d['roofline']['all_hot_loops']: print('   ', h['kernel'], '%.1f ms'%h['ms'], h['launches'], '%.0f GB/s'%h['achieved'])"
  done
done
unset PC_NO_VMARCH
CMD="python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv $CMD > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_vec_march" -s 5 -c 2 -o gpurun_out/${TAG}_vm $CMD > gpurun_out/${TAG}_vm_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_vm.ncu-rep --page raw --csv > gpurun_out/${TAG}_vm_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_vm.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_vm_src.csv 2>/dev/null
ls gpurun_out | head -50
