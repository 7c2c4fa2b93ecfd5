mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/t16.log 2>&1
echo "tests rc=$?" >> gpurun_out/t16.log
L="paper_2407_10449_b200/libtmvn.so"
( for k in 1 2; do REPS=1 PROFILE=0 ITERS=2000 WARM=50 LATENCY=2 python tools/ab_time.py $k 0 1 0 $L; done ) > gpurun_out/ab16.log 2>&1
