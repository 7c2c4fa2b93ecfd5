mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_epi4.so"
( REPS=1 PROFILE=0 PIPE=1 python tools/ab_time.py 3 0 1 0 $L; REPS=1 PROFILE=0 python tools/ab_time.py 3 0 2 0 $L; REPS=1 PROFILE=0 python tools/ab_time.py 3 0 1 0 $L ) > gpurun_out/ab23.log 2>&1
