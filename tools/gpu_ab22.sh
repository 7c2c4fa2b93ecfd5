mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "stages or step or api or moments" > gpurun_out/t22.log 2>&1
echo "tests rc=$?" >> gpurun_out/t22.log
L="paper_2407_10449_b200/libtmvn.so build/libtmvn_c4.so"
( REPS=2 python tools/ab_time.py 3 0 1 0 $L; REPS=1 python tools/ab_time.py 4 0 1 0 $L ) > gpurun_out/ab22.log 2>&1
