# 1 GPU: automatic tile choice test
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "automatic_tile" > gpurun_out/r02mm_tests.log 2>&1; echo rc=$? >> gpurun_out/r02mm_tests.log
