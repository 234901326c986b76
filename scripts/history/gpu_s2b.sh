# bulk-store scatter: parity (single GPU), then N=1 bench both modes, cfg5 size sweep both modes
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s2b_tests.log 2>&1; echo rc=$? >> gpurun_out/s2b_tests.log
for m in threads bulk; do
  timeout 300 python bench.py --steps 10 --warmup 3 --scatter $m --no-e2e --no-cpu-baseline > gpurun_out/s2b_bench_$m.json 2> gpurun_out/s2b_bench_$m.err
  timeout 600 python bench_suite.py cfg5 --scatter $m > gpurun_out/s2b_cfg5_$m.jsonl 2> gpurun_out/s2b_cfg5_$m.err
done
echo done
