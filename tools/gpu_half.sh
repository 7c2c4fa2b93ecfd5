timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/half_t.log 2>&1; echo rc=$? >> gpurun_out/half_t.log
python tools/oz_timing.py 4 10 > gpurun_out/half_oz.log 2>&1
python tools/ab_time.py 4 0 0 0 build/libtmvn_h4.so build/libtmvn_h0.so > gpurun_out/half_ab.log 2>&1
python tools/ab_time.py 4 0 1 0 build/libtmvn_h4.so build/libtmvn_h0.so >> gpurun_out/half_ab.log 2>&1
