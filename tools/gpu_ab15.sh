mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_stg4.so build/libtmvn_stg8.so"
( REPS=1 python tools/ab_time.py 3 0 1 0 $L ) > gpurun_out/ab15.log 2>&1
