SHAPES=1000:200 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so build/libtmvn_force.so > gpurun_out/s42_30.log 2>&1
SHAPES=1000:200 ITERS=1000 BUCKETS=2,0 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so >> gpurun_out/s42_30.log 2>&1
SHAPES=1000:200 ITERS=100 BUCKETS=2,0 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so >> gpurun_out/s42_30.log 2>&1
