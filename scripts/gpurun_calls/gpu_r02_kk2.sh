# 2 GPUs: scan fused into the histogram's last CTA for small forwards -- full GPU suite (world 2), debug parity, latency/sweep/cfg1, bench
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02kk_tests.log 2>&1; echo rc=$? >> gpurun_out/r02kk_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02kk_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02kk_tests_debug.log
for w in latency cfg1 sweep; do timeout 600 python bench_suite.py $w > gpurun_out/r02kk_suite_n1_$w.jsonl 2> gpurun_out/r02kk_suite_n1_$w.err; done
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591"
for w in latency cfg1 sweep; do timeout 600 $RUN2 bench_suite.py $w --gpus 2 > gpurun_out/r02kk_suite_n2_$w.jsonl 2> gpurun_out/r02kk_suite_n2_$w.err; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02kk_bench_n1.json 2> gpurun_out/r02kk_bench_n1.err
echo done
