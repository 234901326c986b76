# 1 GPU: full GPU suite (+debug parity) after the 128-tile warp floor
timeout 1800 python -m pytest tests -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02tt_tests.log 2>&1; echo rc=$? >> gpurun_out/r02tt_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -p no:cacheprovider --timeout 300 > gpurun_out/r02tt_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02tt_tests_debug.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02tt_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02tt_smoke.log
echo done
