mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/t_all.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_all.log
python tools/ab_time.py 3 4,8 1 0 build/libtmvn_cs.so build/libtmvn_pre.so build/libtmvn_pre2.so > gpurun_out/ab.log 2>&1
