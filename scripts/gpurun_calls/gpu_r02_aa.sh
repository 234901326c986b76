# 1 GPU: histogram with two 128-tile scan blocks per 8-KiB stage -- parity (+debug), R=8 sweep 96/128 B
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -m gpu --timeout 300 > gpurun_out/r02aa_tests.log 2>&1; echo rc=$? >> gpurun_out/r02aa_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02aa_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02aa_tests_debug.log
for B in 96 128 48; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02aa_sweep.jsonl 2>&1; done
echo done
