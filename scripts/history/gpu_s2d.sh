# bulk scatter tile sweep (N=1), threads reference
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bulk" > gpurun_out/s2d_tests.log 2>&1; echo rc=$? >> gpurun_out/s2d_tests.log
for T in 256 512 1024 2048; do
  timeout 600 python bench_suite.py cfg5 --scatter bulk --tile $T --sizes 16,24,32,44,48,64,128 > gpurun_out/s2d_bulk_T$T.jsonl 2> gpurun_out/s2d_bulk_T$T.err
done
echo done
