mkdir -p gpurun_out
make -s all > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/t19.log 2>&1
echo "tests rc=$?" >> gpurun_out/t19.log
python bench.py > gpurun_out/bench19.log 2> gpurun_out/bench19.err
