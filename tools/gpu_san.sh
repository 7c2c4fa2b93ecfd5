mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python tools/repro_graph.py > gpurun_out/san.log 2>&1
echo "rc=$?" >> gpurun_out/san.log
