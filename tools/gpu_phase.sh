mkdir -p gpurun_out
for W in 8; do W=$W python tools/phase_timing.py 3 10; done > gpurun_out/phase.log 2>&1
