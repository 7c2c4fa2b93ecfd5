SHAPES=1000:200 python tools/s42_time.py paper_2407_10449_b200/libtmvn.so > gpurun_out/s42_29.log 2>&1
for bk in 1 2 0; do echo "BUCKETS=$bk"; BUCKETS=$bk PAPER_D=1000 PAPER_C=200 python tools/phase_timing.py 3 12; done > gpurun_out/ph29.log 2>&1
