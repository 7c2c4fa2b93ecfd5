mkdir -p gpurun_out
for W in 2 8; do
python tools/ess_one.py 3 $W > gpurun_out/plain_$W.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 3 -c 1 -o gpurun_out/prof_w$W python tools/ess_one.py 3 $W > gpurun_out/ncu_w$W.log 2>&1
done
echo done > gpurun_out/ncu_rc.txt
