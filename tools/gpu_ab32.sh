SHAPES=1000:1000 ITERS=1000 BUCKETS=2,0,2,0 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so > gpurun_out/s42_32.log 2>&1
for bk in 2 0; do echo "BUCKETS=$bk"; BUCKETS=$bk PAPER_D=1000 PAPER_C=1000 python tools/phase_timing.py 3 40; done > gpurun_out/ph32.log 2>&1
