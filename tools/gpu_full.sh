# full GPU suite + short bench (used by gpurun; results under gpurun_out/)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi1.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/rc.txt
