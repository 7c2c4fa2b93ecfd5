mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; echo "tests rc=$?" >> gpurun_out/rc.txt
for c in 1 2 3 4 6; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1
  echo "c$c rc=$?" >> gpurun_out/rc.txt
done
