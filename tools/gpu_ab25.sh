mkdir -p gpurun_out
cp paper_2407_10449_b200/libtmvn.so build/libtmvn_g3.so
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "stages or options_bitwise" > gpurun_out/t25.log 2>&1
echo "tests rc=$?" >> gpurun_out/t25.log
python tools/s42_time.py build/libtmvn_g3.so build/libtmvn_g6.so build/libtmvn_g10.so > gpurun_out/s42_25.log 2>&1
for k in 3 4; do for bk in 1 2 0; do BUCKETS=$bk python tools/ab_time.py $k 0 0 0 build/libtmvn_g3.so build/libtmvn_g10.so; done; done > gpurun_out/ab25.log 2>&1
