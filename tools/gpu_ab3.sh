mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_base.so"
( REPS=1 python tools/ab_time.py 3 0 1 0 $L
  REPS=1 RECORD=0 python tools/ab_time.py 3 0 1 0 $L
  REPS=1 RECORD=0 SCHED=1 python tools/ab_time.py 3 0 1 0 $L
  REPS=1 python tools/ab_time.py 4 0 1 0 $L ) > gpurun_out/ab3.log 2>&1
