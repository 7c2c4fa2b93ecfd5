mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/t13.log 2>&1
echo "tests rc=$?" >> gpurun_out/t13.log
L="paper_2407_10449_b200/libtmvn.so"
( for k in 3 4 5; do REPS=1 OVL=1 python tools/ab_time.py $k 0 1 0 $L; REPS=1 OVL=0 python tools/ab_time.py $k 0 1 0 $L; done
  REPS=1 PROFILE=0 OVL=1 python tools/ab_time.py 3 0 1 0 $L; REPS=1 PROFILE=0 OVL=0 python tools/ab_time.py 3 0 1 0 $L
  ) > gpurun_out/ab13.log 2>&1
