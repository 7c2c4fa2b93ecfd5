# A/B timing of build/libtmvn_$A.so vs build/libtmvn_$B.so on configs $CFGS, then the GPU suite on the in-tree library
mkdir -p gpurun_out
for k in ${CFGS:-3}; do
  python tools/ab_time.py $k 0 0,1 0 build/libtmvn_$A.so build/libtmvn_$B.so >> gpurun_out/ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/ab_t.log 2>&1; echo rc=$? >> gpurun_out/ab_t.log
tail -3 gpurun_out/ab_t.log; cat gpurun_out/ab.log
