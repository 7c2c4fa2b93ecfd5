mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1
echo "rc=$?" >> gpurun_out/bench_full.log
for k in 1 2 4; do python tools/ab_time.py $k 0 1 0 paper_2407_10449_b200/libtmvn.so; done > gpurun_out/other_cfgs.log 2>&1
