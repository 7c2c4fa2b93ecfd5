mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so"
( for S in 1 2 3 4 8; do REPS=1 PROFILE=0 python tools/ab_time.py 3 0 $S 0 $L; done
  for S in 1 2 4; do REPS=1 PROFILE=0 python tools/ab_time.py 5 0 $S 0 $L; done
  for S in 1 2 4; do REPS=1 PROFILE=0 python tools/ab_time.py 4 0 $S 0 $L; done ) > gpurun_out/ab18.log 2>&1
