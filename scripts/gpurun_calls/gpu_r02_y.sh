# 1 GPU: cfg5 as configs[4] -- 8 ranks x 32M items (8 logical ranks), sizes 16..128 B
timeout 1500 python bench_suite.py cfg5 > gpurun_out/r02y_cfg5_r8_n1.jsonl 2> gpurun_out/r02y_cfg5_r8_n1.err
echo done
