# 1 GPU: full-size cfg3 / cfg4 against the sampled CPU twin
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "cfg3 or cfg4" --timeout 900 --durations=5 > gpurun_out/r02ee_tests.log 2>&1; echo rc=$? >> gpurun_out/r02ee_tests.log
echo done
