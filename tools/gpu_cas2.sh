python tools/ab_time.py 4 0 0 0 build/libtmvn_c1.so build/libtmvn_c0.so > gpurun_out/cas2.log 2>&1
ITERS=3 WARM=2 python tools/ab_time.py 5 0 0 0 build/libtmvn_c1.so build/libtmvn_c0.so >> gpurun_out/cas2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/cas2_t.log 2>&1; echo rc=$? >> gpurun_out/cas2_t.log
