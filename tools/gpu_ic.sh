for k in 3 4; do for v in 2 1; do echo "cfg $k variant $v"; TIMING_LIB=build/libtmvn_tim$v.so python tools/oz_timing.py $k 10; done; done > gpurun_out/ic_oz.log 2>&1
for k in 3 4; do python tools/ab_time.py $k 0 0 0 build/libtmvn_ic2.so build/libtmvn_ic1.so; done > gpurun_out/ic_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_step.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > gpurun_out/ic_t.log 2>&1; echo rc=$? >> gpurun_out/ic_t.log
