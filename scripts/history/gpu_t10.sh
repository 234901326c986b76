timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench10_n1.json 2> gpurun_out/bench10_n1.err
timeout 300 python bench_suite.py cfg5 > gpurun_out/cfg5_10.jsonl 2>&1
