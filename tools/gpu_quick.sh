mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/t_all.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_all.log
python tools/ab_time.py 3 2 1,2 0 paper_2407_10449_b200/libtmvn.so > gpurun_out/ab.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
