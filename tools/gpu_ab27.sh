mkdir -p gpurun_out
python tools/s42_time.py paper_2407_10449_b200/libtmvn.so > gpurun_out/s42_27.log 2>&1
for k in 3 4; do for bk in 1 0; do BUCKETS=$bk python tools/ab_time.py $k 0 0 0 paper_2407_10449_b200/libtmvn.so; done; done > gpurun_out/ab27.log 2>&1
( PAPER_D=1000 PAPER_C=200 python tools/phase_timing.py 3 12 ) > gpurun_out/ph27.log 2>&1
