mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_step.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_oz.log 2>&1
echo "oz tests rc=$?" >> gpurun_out/rc.txt
timeout 200 python tools/oz_timing.py 3 10 > gpurun_out/oz_timing.log 2>&1
echo "oz timing rc=$?" >> gpurun_out/rc.txt
PROFILE=1 timeout 300 python tools/ab_time.py 3 0 1 0 paper_2407_10449_b200/libtmvn.so > gpurun_out/ab.log 2>&1
PROFILE=0 timeout 300 python tools/ab_time.py 3 0 1 0 paper_2407_10449_b200/libtmvn.so >> gpurun_out/ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/rc.txt
