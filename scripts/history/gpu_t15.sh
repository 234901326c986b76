timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench15_n1.json 2> gpurun_out/bench15_n1.err
timeout 300 python bench_suite.py sweep > gpurun_out/sweep15.jsonl 2>&1
