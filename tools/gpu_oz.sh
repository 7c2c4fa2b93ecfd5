# int8 tcgen05 projection: tests + short benches (results under gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_oz.log 2>&1
echo "oz tests rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --projection 1 > gpurun_out/bench_oz.log 2>&1
echo "bench oz rc=$?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/rc.txt
