python tools/ab_time.py 4 0 0 0 build/libtmvn_aq1.so build/libtmvn_aq0.so > gpurun_out/aq.log 2>&1
python tools/ab_time.py 4 16 1 0 build/libtmvn_aq1.so build/libtmvn_aq0.so >> gpurun_out/aq.log 2>&1
ITERS=3 WARM=2 python tools/ab_time.py 5 0 0 0 build/libtmvn_aq1.so build/libtmvn_aq0.so >> gpurun_out/aq.log 2>&1
python tools/ab_time.py 3 0 0 0 build/libtmvn_aq1.so build/libtmvn_aq0.so >> gpurun_out/aq.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/aq_t.log 2>&1; echo rc=$? >> gpurun_out/aq_t.log
