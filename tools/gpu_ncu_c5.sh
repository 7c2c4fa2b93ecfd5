mkdir -p gpurun_out
for pr in 1 2; do
CMD="python bench.py --config 5 --steps 1 --warmup 1 --iters-per-step 2 --no-cpu-baseline --no-e2e --projection $pr"
$CMD > gpurun_out/plain_$pr.log 2>&1 &&
ncu --set full --clock-control none -k regex:ess_kernel -s 2 -c 1 -o gpurun_out/prof_c5_$pr $CMD > gpurun_out/ncu_c5_$pr.log 2>&1
echo "pr$pr rc=$?" >> gpurun_out/ncu_rc.txt
done
