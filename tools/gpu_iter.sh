# iterate: full GPU tests, ESS phase timing, short bench (results under gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/rc.txt
timeout 200 python tools/phase_timing.py 3 10 > gpurun_out/phase.log 2>&1
echo "phase rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/rc.txt
