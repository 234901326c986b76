# aligned (16-B thread stores after the smem permutation) vs threads vs bulk, N=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s2f_tests.log 2>&1; echo rc=$? >> gpurun_out/s2f_tests.log
for m in aligned threads bulk; do
  timeout 600 python bench_suite.py cfg5 --scatter $m > gpurun_out/s2f_cfg5_$m.jsonl 2> gpurun_out/s2f_cfg5_$m.err
done
for T in 256 512 1024; do
  timeout 600 python bench_suite.py cfg5 --scatter aligned --tile $T --sizes 16,24,32,44,48,64,128 > gpurun_out/s2f_al_T$T.jsonl 2> gpurun_out/s2f_al_T$T.err
done
echo done
