# 2 GPUs: nibble-counter histogram + file rendezvous in the multi-process tests -- full GPU suite (world 2), debug parity, hist sweep
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02gg_tests.log 2>&1; echo rc=$? >> gpurun_out/r02gg_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02gg_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02gg_tests_debug.log
for B in 48 64 128 16; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02gg_sweep.jsonl 2>&1; done
timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 16777216 >> gpurun_out/r02gg_sweep.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02gg_bench_n1.json 2> gpurun_out/r02gg_bench_n1.err
echo done
