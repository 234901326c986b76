# 1 GPU: parity after the hist fast path; bench N=1; ncu of k_hist
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_nbody.py tests/test_streamlines.py tests/test_proxies.py -x -q > gpurun_out/s3f_tests.log 2>&1; echo rc=$? >> gpurun_out/s3f_tests.log
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/s3f_bench_n1.json 2> gpurun_out/s3f_bench_n1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3f_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_hist" -s 2 -c 1 -o gpurun_out/s3f_hist python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3f_ncu.log 2>&1
echo done
