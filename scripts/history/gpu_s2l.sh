# 1 GPU: parity with the 16-B chunk gather, cfg5 threads (chunk) vs units
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2l_tests.log 2>&1; echo rc=$? >> gpurun_out/s2l_tests.log
for m in threads units; do
  timeout 600 python bench_suite.py cfg5 --scatter $m > gpurun_out/s2l_cfg5_$m.jsonl 2> gpurun_out/s2l_cfg5_$m.err
done
python bench.py --steps 10 --warmup 3 > gpurun_out/s2l_bench_n1.json 2> gpurun_out/s2l_bench_n1.err
echo done
