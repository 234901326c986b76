# 1 GPU: per-size TMA stages in the warp scatter -- full GPU suite (+debug parity), R=8 size sweep, bench
timeout 1800 python -m pytest tests -x -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02ss_tests.log 2>&1; echo rc=$? >> gpurun_out/r02ss_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02ss_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02ss_tests_debug.log
for B in 16 20 24 32 40 44 48 64 96 128; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02ss_sweep.jsonl 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02ss_bench_n1.json 2> gpurun_out/r02ss_bench_n1.err
echo done
