mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1
echo "rc=$?" >> gpurun_out/bench_full.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo "rc=$?" >> gpurun_out/bench_ref.log
