for k in 3 2; do python tools/ab_time.py $k 0 0 0 build/libtmvn_p1.so build/libtmvn_p0.so; done > gpurun_out/p.log 2>&1
SHAPES=1000:200,1000:1000 BUCKETS=0 python tools/s42_time.py build/libtmvn_p1.so build/libtmvn_p0.so >> gpurun_out/p.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/p_t.log 2>&1; echo rc=$? >> gpurun_out/p_t.log
