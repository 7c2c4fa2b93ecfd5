# config 4: isolated kernel times (one shard), projection role timing, per-chain phases
mkdir -p gpurun_out
make -s timing > /dev/null 2>&1
( python tools/ab_time.py 4 0 1,4 0 paper_2407_10449_b200/libtmvn.so ) > gpurun_out/c4_ab.log 2>&1
( python tools/oz_timing.py 4 10 ) > gpurun_out/c4_oz.log 2>&1
( python tools/phase_timing.py 4 5 ) > gpurun_out/c4_ph.log 2>&1
