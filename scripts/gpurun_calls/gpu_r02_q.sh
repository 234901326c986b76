# 1 GPU: chunk gather with 16-B shared windows -- parity (+debug), R=8 sweep (chunk vs 8-B units)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_proxies.py -x -q -p no:cacheprovider -m gpu --timeout 300 > gpurun_out/r02q_tests.log 2>&1; echo rc=$? >> gpurun_out/r02q_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02q_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02q_tests_debug.log
for B in 44 20 12 40 24; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02q_sweep.jsonl 2>&1; done
for B in 40 24; do RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_c8off.so timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02q_sweep_c8off.jsonl 2>&1; done
echo done
