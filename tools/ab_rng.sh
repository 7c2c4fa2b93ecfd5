mkdir -p gpurun_out
for r in 1 2; do for ra in 0 1; do RNG_AHEAD=$ra PROFILE=0 REPS=1 timeout 200 python tools/ab_time.py 3 0 1 0 paper_2407_10449_b200/libtmvn.so; done; done > gpurun_out/ab.log 2>&1
