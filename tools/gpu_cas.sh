for k in 3 4; do python tools/ab_time.py $k 0 0 0 build/libtmvn_cas1.so build/libtmvn_cas0.so; done > gpurun_out/cas_ab.log 2>&1
SHAPES=1000:1000,1000:200 BUCKETS=0 python tools/s42_time.py build/libtmvn_cas1.so build/libtmvn_cas0.so > gpurun_out/cas_s42.log 2>&1
