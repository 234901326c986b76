timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_proxies.py -x -q > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench9_n1.json 2> gpurun_out/bench9_n1.err
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --item-bytes 44 > gpurun_out/bench9_b44.json 2> gpurun_out/bench9_b44.err
timeout 300 python bench_suite.py cfg5 > gpurun_out/cfg5_9.jsonl 2>&1
timeout 300 python bench_suite.py latency > gpurun_out/lat9.jsonl 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat9_launches.csv python bench_suite.py latency > gpurun_out/lat9_ncu.log 2>&1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --item-bytes 44 > gpurun_out/plain44.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_scatter -s 2 -c 1 -o gpurun_out/prof_scatter44 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --item-bytes 44 > gpurun_out/ncu44.log 2>&1
