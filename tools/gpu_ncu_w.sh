mkdir -p gpurun_out
python tools/ess_one.py 3 8 > gpurun_out/plain_8.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ess_kernel -s 3 -c 1 -o gpurun_out/prof_w8b python tools/ess_one.py 3 8 > gpurun_out/ncu_w8.log 2>&1
echo done > gpurun_out/ncu_rc.txt
