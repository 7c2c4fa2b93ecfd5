mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi1.txt
timeout 400 python -m pytest tests/test_gpu_stages.py -q --timeout 300 -p no:cacheprovider > gpurun_out/t_stages.log 2>&1
echo "stages rc=$?" >> gpurun_out/rc.txt
timeout 700 python -m pytest tests/test_gpu_step.py -q --timeout 400 -p no:cacheprovider > gpurun_out/t_step.log 2>&1
echo "step rc=$?" >> gpurun_out/rc.txt
timeout 700 python -m pytest tests/test_gpu_api.py -q --timeout 400 -p no:cacheprovider > gpurun_out/t_api.log 2>&1
echo "api rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/rc.txt
