mkdir -p gpurun_out
make -s all > /dev/null 2>&1
( REPS=1 python tools/ab_time.py 3 0 1 0 paper_2407_10449_b200/libtmvn.so build/libtmvn_nornd.so ) > gpurun_out/ab8.log 2>&1
