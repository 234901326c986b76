# 4 GPUs: cfg5 (8 ranks) write path at N=2/4 -- warp-tile THREADS vs BULK, per item size
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562"
timeout 900 $RUN2 bench_suite.py cfg5 --gpus 2 --scatter threads --sizes 16,24,32,44,48,64,128 > gpurun_out/r02bb_cfg5_n2_threads.jsonl 2> gpurun_out/r02bb_cfg5_n2_threads.err
timeout 900 $RUN4 bench_suite.py cfg5 --gpus 4 --scatter threads --sizes 16,24,32,44,48,64,128 > gpurun_out/r02bb_cfg5_n4_threads.jsonl 2> gpurun_out/r02bb_cfg5_n4_threads.err
echo done
