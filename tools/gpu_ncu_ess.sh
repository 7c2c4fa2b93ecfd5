# full ncu capture of the fused ESS kernel only
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --iters-per-step 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 3 -c 1 -o gpurun_out/prof_ess4 $CMD > gpurun_out/ncu_ess.log 2>&1
echo "rc=$?" > gpurun_out/ncu_rc.txt
