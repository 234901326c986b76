# 1 GPU: parity after the emit fast path + dest prefetch; bench N=1; cfg5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2x_tests.log 2>&1; echo rc=$? >> gpurun_out/s2x_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s2x_bench_n1.json 2> gpurun_out/s2x_bench_n1.err
timeout 600 python bench_suite.py cfg5 > gpurun_out/s2x_cfg5.jsonl 2> gpurun_out/s2x_cfg5.err
echo done
