mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_step.py tests/test_gpu_api.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/t_all.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_all.log
python tools/ab_time.py 3 2,4,8 1,2 0,1 build/libtmvn_mb2.so build/libtmvn_mb3.so > gpurun_out/ab.log 2>&1
