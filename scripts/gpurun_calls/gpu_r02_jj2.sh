# 2 GPUs: single-process peer redirect test
timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider -k "redirect" --timeout 300 > gpurun_out/r02jj_tests.log 2>&1; echo rc=$? >> gpurun_out/r02jj_tests.log
echo done
