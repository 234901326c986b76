timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_nbody.py -x -q > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench13_n1.json 2> gpurun_out/bench13_n1.err
timeout 300 python bench_suite.py cfg5 > gpurun_out/cfg5_13.jsonl 2>&1
timeout 300 python bench_suite.py sweep > gpurun_out/sweep13.jsonl 2>&1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain13.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches13.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu13a.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_hist" -s 2 -c 2 -o gpurun_out/prof13 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu13b.log 2>&1
