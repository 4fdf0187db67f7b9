# experiment: k_pcg_pupdatev variants (pairs per lane, blocks per SM) on C4, ncu launch times
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --config c4 --steps 1 --warmup 0"
for V in 0 1 2; do
  PC_PUPD=$V timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pcg_pupdatev -c 12 --csv --log-file gpurun_out/pupd_$V.csv $B > /dev/null 2>&1
  echo "variant $V"; python scripts/ncu_launches.py gpurun_out/pupd_$V.csv 2>/dev/null | sed -n 2p
done
