mkdir -p gpurun_out/fin
make -s all > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/fin/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/fin/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/fin/smoke.log
python bench.py > gpurun_out/fin/bench.jsonl 2> gpurun_out/fin/bench.err
echo "rc=$?" >> gpurun_out/fin/bench.err
