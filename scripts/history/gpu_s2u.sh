# 1 GPU: cfg5 threads (16-B chunk gather) vs units; bench N=1; sweep (44 B)
for m in threads units; do
  timeout 600 python bench_suite.py cfg5 --scatter $m > gpurun_out/s2u_cfg5_$m.jsonl 2> gpurun_out/s2u_cfg5_$m.err
done
python bench.py --steps 10 --warmup 3 > gpurun_out/s2u_bench_n1.json 2> gpurun_out/s2u_bench_n1.err
timeout 300 python bench_suite.py sweep > gpurun_out/s2u_sweep.jsonl 2> gpurun_out/s2u_sweep.err
echo done
