timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s4d_tests.log 2>&1; echo rc=$? >> gpurun_out/s4d_tests.log
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/s4d_bench_n1.json 2> gpurun_out/s4d_bench_n1.err
timeout 600 python bench_suite.py cfg5 --sizes 44,48,64,128 > gpurun_out/s4d_cfg5.jsonl 2> gpurun_out/s4d_cfg5.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4d_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4d_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4d_ncu.log 2>&1
echo done
