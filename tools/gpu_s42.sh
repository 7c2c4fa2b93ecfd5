mkdir -p gpurun_out
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/bench_c6.log 2>&1; echo "c6 rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 --projection 2 --no-cpu-baseline > gpurun_out/bench_c6_dmma.log 2>&1; echo "c6d rc=$?" >> gpurun_out/rc.txt
