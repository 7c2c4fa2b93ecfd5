# round evidence: default bench (cpu baseline + e2e), reference arm, smoke, launch list, ncu full of the two hot kernels
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
CMD="python bench.py --steps 1 --warmup 1 --iters-per-step 40 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 4 -c 1 -o gpurun_out/prof_oz $CMD > gpurun_out/ncu_oz.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 4 -c 1 -o gpurun_out/prof_ess $CMD > gpurun_out/ncu_ess.log 2>&1
echo "ncu rc=$?" >> gpurun_out/rc.txt
# the other workloads (latency mode, FP32-class, configs 4/5)
timeout 600 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/bench_c6.log 2>&1; echo "c6 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --config 7 --steps 3 --warmup 3 > gpurun_out/bench_c7.log 2>&1; echo "c7 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --precision 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1; echo "fp32 rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --iters-per-step 20 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/rc.txt
