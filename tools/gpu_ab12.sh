mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so"
( for k in 2 1; do REPS=1 PROFILE=0 ITERS=500 WARM=50 LATENCY=1 python tools/ab_time.py $k 0 1 0 $L; REPS=1 PROFILE=0 ITERS=500 WARM=50 LATENCY=0 python tools/ab_time.py $k 0 1 0 $L; REPS=1 PROFILE=0 ITERS=500 WARM=50 LATENCY=2 python tools/ab_time.py $k 0 1 0 $L; done ) > gpurun_out/ab12.log 2>&1
