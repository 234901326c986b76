# 4 GPUs: bench N=1/2/4 on the fixed bench (no NVML in the timed region), multi-GPU parity at world 2 and 4
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522"
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r02k_bench_n1.json 2> gpurun_out/r02k_bench_n1.err
$RUN2 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k_bench_n2.json 2> gpurun_out/r02k_bench_n2.err
$RUN4 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k_bench_n4.json 2> gpurun_out/r02k_bench_n4.err
$RUN4 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --scatter threads > gpurun_out/r02k_bench_n4_threads.json 2> gpurun_out/r02k_bench_n4_threads.err
timeout 1800 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/r02k_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02k_multiproc.log
echo done
