mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_band16.so build/libtmvn_band32.so build/libtmvn_band4.so"
( REPS=1 ITERS=6 WARM=2 python tools/ab_time.py 5 0 0 0 $L; REPS=1 python tools/ab_time.py 3 0 1 0 $L ) > gpurun_out/ab21.log 2>&1
