mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/san_run.py > gpurun_out/san_mem.log 2>&1
echo "rc=$?" >> gpurun_out/san_mem.log
