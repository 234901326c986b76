# 1 GPU: parity after the hist rewrite, bench N=1, PCIe ceilings, threads-scatter tile sweep
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2k_tests.log 2>&1; echo rc=$? >> gpurun_out/s2k_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s2k_bench_n1.json 2> gpurun_out/s2k_bench_n1.err
timeout 120 ./tools/p2p_bw > gpurun_out/s2k_p2p_n1.jsonl 2>&1
for T in 256 512 1024 2048; do
  timeout 600 python bench_suite.py cfg5 --scatter threads --tile $T --sizes 16,24,32,44,48 > gpurun_out/s2k_thr_T$T.jsonl 2> gpurun_out/s2k_thr_T$T.err
done
echo done
