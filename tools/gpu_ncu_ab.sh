# DRAM bytes and duration per ess_kernel / ozaki launch (config $CFG, one shard) for library variants $LIBS
mkdir -p gpurun_out
cp paper_2407_10449_b200/libtmvn.so /tmp/libtmvn_orig.so
for v in $LIBS; do
  cp build/libtmvn_$v.so paper_2407_10449_b200/libtmvn.so
  BK="python bench.py --config ${CFG:-3} --steps 1 --warmup 1 --iters-per-step 4 --sub-configs= --no-cpu-baseline --no-e2e --streams 1"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:"ess_kernel|ozaki_gemm_kernel" -s 6 -c 6 --csv $BK > gpurun_out/ncu_ab_$v.csv 2> gpurun_out/ncu_ab_$v.err
  echo "$v rc=$?"
done
cp /tmp/libtmvn_orig.so paper_2407_10449_b200/libtmvn.so
