# 1 GPU: final write-path choice per item size -- full single-GPU suite (+debug parity), R=8 sweep of every synthetic size
timeout 1800 python -m pytest tests -x -q -p no:cacheprovider -m gpu --timeout 600 > gpurun_out/r02r_tests.log 2>&1; echo rc=$? >> gpurun_out/r02r_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02r_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02r_tests_debug.log
for B in 4 12 16 20 24 32 40 44 48 64 96 128; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02r_sweep.jsonl 2>&1; done
echo done
