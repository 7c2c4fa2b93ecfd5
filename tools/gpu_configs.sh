mkdir -p gpurun_out
for c in 1 2 4; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1
  echo "c$c rc=$?" >> gpurun_out/rc.txt
done
timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --iters-per-step 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --iters-per-step 4 --no-cpu-baseline --no-e2e --projection 2 > gpurun_out/bench_c5_dmma.log 2>&1
echo "c5 dmma rc=$?" >> gpurun_out/rc.txt
