# 1 GPU: 4-byte-unit warp tiles (B % 8 == 4) -- parity (+debug), R=8 sweep warp vs block tiles
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py tests/test_proxies.py tests/test_nbody.py tests/test_streamlines.py -x -q -p no:cacheprovider -m gpu --timeout 300 > gpurun_out/r02o_tests.log 2>&1; echo rc=$? >> gpurun_out/r02o_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02o_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02o_tests_debug.log
for B in 44 20 12 40 4; do timeout 300 python scripts/prof_binning.py --tiles 0,512,1024,2048 --scatter threads --B $B >> gpurun_out/r02o_sweep.jsonl 2>&1; done
echo done
