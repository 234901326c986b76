# 1 GPU: parity with graph/untimed split; bench N=1; sweep; latency; cfg1; cfg4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q > gpurun_out/s3i_tests.log 2>&1; echo rc=$? >> gpurun_out/s3i_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s3i_bench_n1.json 2> gpurun_out/s3i_bench_n1.err
for w in sweep latency cfg1 cfg4 cfg3; do timeout 600 python bench_suite.py $w > gpurun_out/s3i_$w.jsonl 2> gpurun_out/s3i_$w.err; done
echo done
