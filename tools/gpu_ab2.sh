mkdir -p gpurun_out
make -s all > /dev/null 2>&1
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_base.so"
( python tools/ab_time.py 3 0 1 0 $L
  RECORD=0 python tools/ab_time.py 3 0 1 0 $L
  python tools/ab_time.py 4 0 1 0 $L
  python tools/ab_time.py 2 0 1 0 $L ) > gpurun_out/ab2.log 2>&1
