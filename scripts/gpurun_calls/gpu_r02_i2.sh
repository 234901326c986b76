# 2 GPUs: NVLink counter probes, multi-GPU parity, N=2 bench (bulk vs threads), rank-0 NVLink counters
(nvidia-smi nvlink -s -i 0; nvidia-smi nvlink -gt d -i 0; nvidia-smi topo -m) > gpurun_out/r02i_nvl_probe.txt 2>&1
ncu --query-metrics 2>&1 | grep -i "nvltx\|nvlrx" > gpurun_out/r02i_nvl_metrics.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r02i_nvl_before.txt 2>&1
$RUN bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02i_bench_n2_auto.json 2> gpurun_out/r02i_bench_n2_auto.err
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r02i_nvl_after.txt 2>&1
$RUN bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --scatter threads > gpurun_out/r02i_bench_n2_threads.json 2> gpurun_out/r02i_bench_n2_threads.err
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/r02i_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02i_multiproc.log
timeout 300 $RUN --no-python bash scripts/ncu_rank0.sh gpurun_out/r02i_nvl_ncu_threads.csv bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras --control nccl --scatter threads > gpurun_out/r02i_ncu_threads.log 2>&1; echo rc=$? >> gpurun_out/r02i_ncu_threads.log
timeout 300 $RUN --no-python bash scripts/ncu_rank0.sh gpurun_out/r02i_nvl_ncu_bulk.csv bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras --control nccl --scatter bulk > gpurun_out/r02i_ncu_bulk.log 2>&1; echo rc=$? >> gpurun_out/r02i_ncu_bulk.log
timeout 300 $RUN --no-python bash scripts/ncu_rank0.sh gpurun_out/r02i_nvl_ncu_peer.csv bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras --control nccl --exchange peer > gpurun_out/r02i_ncu_peer.log 2>&1; echo rc=$? >> gpurun_out/r02i_ncu_peer.log
echo done
