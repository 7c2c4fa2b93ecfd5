mkdir -p gpurun_out/r02b
make -s all > /dev/null 2>&1
python bench.py > gpurun_out/r02b/bench.jsonl 2> gpurun_out/r02b/bench.err
echo "rc=$?" >> gpurun_out/r02b/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b/bench_reference.jsonl 2> gpurun_out/r02b/bench_reference.err
python bench.py --precision 1 --sub-configs= > gpurun_out/r02b/bench_fp32_class.jsonl 2>> gpurun_out/r02b/bench.err
python bench.py --config 6 --sub-configs= > gpurun_out/r02b/bench_paper_s42.jsonl 2>> gpurun_out/r02b/bench.err
python bench.py --config 7 --sub-configs= --steps 3 > gpurun_out/r02b/bench_paper_s42_single_d4000.jsonl 2>> gpurun_out/r02b/bench.err
python bench.py --config 5 --sub-configs= --steps 3 --no-e2e > gpurun_out/r02b/bench_config5.jsonl 2>> gpurun_out/r02b/bench.err
python bench.py --projection 2 --sub-configs= > gpurun_out/r02b/bench_fp64_dmma.jsonl 2>> gpurun_out/r02b/bench.err
echo done >> gpurun_out/r02b/bench.err
