timeout 900 python -m pytest tests/test_nbody.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_proxies.py -x -q > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
timeout 300 python bench_suite.py nbody > gpurun_out/nbody11.jsonl 2>&1
