mkdir -p gpurun_out
python tools/ab_time.py 3 2,4,8 1,2 0,1 build/libtmvn_cs.so > gpurun_out/ab.log 2>&1
