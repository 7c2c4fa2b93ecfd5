# round-2 profile set: launch list of the bench command (config 3, default options), ncu
# --set full of the two hot kernels at configs 3 and 4 with one shard (reports kept on the
# box's /tmp; summaries exported)
mkdir -p gpurun_out/r02 /tmp/r02
make -s all > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 1 --sub-configs= --no-cpu-baseline --no-e2e"
$B > gpurun_out/r02/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02/ncu_launches_config3.csv $B > gpurun_out/r02/ncu_launches.log 2>&1
for k in 3 4; do
  # --streams 1: one launch per kernel over all chains (the bench roofline's launch), so the
  # captured DRAM bytes compare with its algorithmic bytes per launch
  BK="python bench.py --config $k --steps 1 --warmup 1 --iters-per-step 4 --sub-configs= --no-cpu-baseline --no-e2e --streams 1"
  ncu --set full --clock-control none --import-source on -f -k regex:"ess_kernel|ozaki_gemm_kernel" -s 6 -c 2 \
      -o /tmp/r02/full_config$k $BK > gpurun_out/r02/ncu_full_config$k.log 2>&1
  ncu -i /tmp/r02/full_config$k.ncu-rep --page raw --csv > gpurun_out/r02/full_config${k}_raw.csv 2>/dev/null
  ncu -i /tmp/r02/full_config$k.ncu-rep --page details --csv > gpurun_out/r02/full_config${k}_details.csv 2>/dev/null
done
python tools/ncu_inst.py /tmp/r02/full_config3.ncu-rep 60 > gpurun_out/r02/ess_inst_config3.txt 2>&1
ls -la /tmp/r02 > gpurun_out/r02/reports.txt
echo done > gpurun_out/r02/rc.txt
