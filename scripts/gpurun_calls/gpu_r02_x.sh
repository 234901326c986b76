# 1 GPU: the other configs on the round-2 kernels (8-rank configs as 8 logical ranks)
for w in cfg1 cfg3 cfg4 cfg5 sweep latency nbody streamlines; do timeout 900 python bench_suite.py $w > gpurun_out/r02x_suite_$w.jsonl 2> gpurun_out/r02x_suite_$w.err; done
echo done
