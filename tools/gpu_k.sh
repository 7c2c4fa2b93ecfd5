python tools/ab_time.py 4 0 0 0 build/libtmvn_k1.so build/libtmvn_k0.so > gpurun_out/k.log 2>&1
ITERS=3 WARM=2 python tools/ab_time.py 5 0 0 0 build/libtmvn_k1.so build/libtmvn_k0.so >> gpurun_out/k.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/k_t.log 2>&1; echo rc=$? >> gpurun_out/k_t.log
