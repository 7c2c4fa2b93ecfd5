mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/t26.log 2>&1
echo "tests rc=$?" >> gpurun_out/t26.log
python tools/s42_time.py paper_2407_10449_b200/libtmvn.so > gpurun_out/s42_26.log 2>&1
for k in 3 4; do for bk in 1 0; do BUCKETS=$bk python tools/ab_time.py $k 0 0 0 paper_2407_10449_b200/libtmvn.so; done; done > gpurun_out/ab26.log 2>&1
