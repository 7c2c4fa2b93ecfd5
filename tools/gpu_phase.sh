mkdir -p gpurun_out
for k in 3 2 4; do python tools/phase_timing.py $k 10; done > gpurun_out/phase.log 2>&1
