# round-1 evidence: launch list of the bench command, full captures of the two hot kernels
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --iters-per-step 40 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 4 -c 1 -o gpurun_out/prof_oz $CMD > gpurun_out/ncu_oz.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 4 -c 1 -o gpurun_out/prof_ess $CMD > gpurun_out/ncu_ess.log 2>&1
echo "rc=$?" > gpurun_out/ncu_rc.txt
