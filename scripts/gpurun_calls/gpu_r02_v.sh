# 1 GPU: run tracking back for 16-B units; 44 B chunk vs 4-B units -- parity (+debug), R=8 sweep, bench
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -m gpu --timeout 300 > gpurun_out/r02v_tests.log 2>&1; echo rc=$? >> gpurun_out/r02v_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02v_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02v_tests_debug.log
for B in 16 20 24 32 40 44 48 64; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02v_sweep.jsonl 2>&1; done
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_nochunk.so timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 44 >> gpurun_out/r02v_sweep_nochunk.jsonl 2>&1
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_nochunk.so timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 44 --L 1 --n 134217728 >> gpurun_out/r02v_sweep_nochunk.jsonl 2>&1
timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 44 --L 1 --n 134217728 >> gpurun_out/r02v_sweep.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02v_bench_n1.json 2> gpurun_out/r02v_bench_n1.err
echo done
