mkdir -p gpurun_out
( timeout 60 ./tools/tc_i8_gemm 128 256 256; echo "rc=$?"; timeout 60 ./tools/tc_i8_gemm 4096 2048 1024; echo "rc=$?" ) > gpurun_out/tc.log 2>&1
