# round 2: the GPU suite (all failures reported), with durations and printed logs
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_gpu.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_gpu.log
tail -5 gpurun_out/t_gpu.log
