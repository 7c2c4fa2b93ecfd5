SHAPES=1000:200,1000:1000,600:400 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so > gpurun_out/s42_31.log 2>&1
for k in 3 4; do for bk in 1 0; do BUCKETS=$bk python tools/ab_time.py $k 0 0 0 paper_2407_10449_b200/libtmvn.so; done; done > gpurun_out/ab31.log 2>&1
