# 2 GPUs: small rounds with warp tiles (hist+scan fused) vs BULK at N=2
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592"
timeout 600 $RUN2 bench_suite.py sweep --gpus 2 --scatter threads > gpurun_out/r02ll_sweep_n2_threads.jsonl 2> gpurun_out/r02ll_sweep_n2_threads.err
timeout 600 $RUN2 bench_suite.py latency --gpus 2 --scatter threads > gpurun_out/r02ll_latency_n2_threads.jsonl 2> gpurun_out/r02ll_latency_n2_threads.err
echo done
