mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --iters-per-step 8 --no-cpu-baseline --no-e2e --sub-configs="
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 3 -c 1 -o gpurun_out/prof_ess_${TAG:-x} $CMD > gpurun_out/ncu_ess.log 2>&1
echo "rc=$?" > gpurun_out/ncu_rc.txt
python tools/ncu_inst.py gpurun_out/prof_ess_${TAG:-x}.ncu-rep 120 > gpurun_out/ess_inst_${TAG:-x}.txt 2>&1
