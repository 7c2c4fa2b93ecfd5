mkdir -p gpurun_out
make -s all > /dev/null 2>&1
t0=$(date +%s)
python bench.py $BENCH_ARGS > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/bench.err
