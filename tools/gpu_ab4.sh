mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t4.log 2>&1
echo "tests rc=$?" >> gpurun_out/t4.log
L="paper_2407_10449_b200/libtmvn.so"
( REPS=1 FUSE=1 python tools/ab_time.py 3 0 1 0 $L
  REPS=1 FUSE=0 python tools/ab_time.py 3 0 1 0 $L
  REPS=1 python tools/ab_time.py 3 0 1 0 build/libtmvn_base.so
  REPS=1 FUSE=1 python tools/ab_time.py 4 0 1 0 $L
  REPS=1 FUSE=0 python tools/ab_time.py 4 0 1 0 $L
  REPS=1 FUSE=1 python tools/ab_time.py 5 0 1 0 $L
  REPS=1 FUSE=0 python tools/ab_time.py 5 0 1 0 $L
  REPS=1 FUSE=1 python tools/ab_time.py 2 0 1 0 $L
  REPS=1 FUSE=0 python tools/ab_time.py 2 0 1 0 $L
  ) > gpurun_out/ab4.log 2>&1
