# 1 GPU then 2 GPUs: the bench with its supplementary graph-replay line
python bench.py > gpurun_out/s4f_bench_n1.json 2> gpurun_out/s4f_bench_n1.err
python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 > gpurun_out/s4f_bench_n2.json 2> gpurun_out/s4f_bench_n2.err
echo done
