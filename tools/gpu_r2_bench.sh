# round 2: selected GPU tests + the default bench line (+ a 2-GPU-plumbing dry check is CPU-only)
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_sel.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_sel.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
