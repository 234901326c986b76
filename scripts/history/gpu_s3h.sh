# 1 GPU: parity with the cached forward graph; sweep/latency A/B graph on/off; bench N=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_nbody.py tests/test_streamlines.py tests/test_proxies.py -x -q > gpurun_out/s3h_tests.log 2>&1; echo rc=$? >> gpurun_out/s3h_tests.log
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/s3h_bench_n1.json 2> gpurun_out/s3h_bench_n1.err
timeout 600 python bench_suite.py sweep > gpurun_out/s3h_sweep.jsonl 2> gpurun_out/s3h_sweep.err
timeout 600 python bench_suite.py latency > gpurun_out/s3h_lat.jsonl 2> gpurun_out/s3h_lat.err
timeout 600 python bench_suite.py cfg1 > gpurun_out/s3h_cfg1.jsonl 2> gpurun_out/s3h_cfg1.err
timeout 600 python bench_suite.py cfg4 > gpurun_out/s3h_cfg4.jsonl 2> gpurun_out/s3h_cfg4.err
echo done
