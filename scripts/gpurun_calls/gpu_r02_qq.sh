# 1 GPU: histogram 12 warps x 1 stage (256) / 16 x 1 (128) -- parity (+debug), sweep, bench
timeout 1800 python -m pytest tests -x -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02qq_tests.log 2>&1; echo rc=$? >> gpurun_out/r02qq_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02qq_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02qq_tests_debug.log
for B in 16 48 64 96 128; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02qq_sweep.jsonl 2>&1; done
timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 16777216 >> gpurun_out/r02qq_sweep.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02qq_bench_n1.json 2> gpurun_out/r02qq_bench_n1.err
timeout 600 python bench_suite.py latency > gpurun_out/r02qq_latency.jsonl 2> gpurun_out/r02qq_latency.err
echo done
