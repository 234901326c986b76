# 2 GPUs: final tree multi-GPU parity (world 2) + bench N=2
timeout 1800 python -m pytest tests/test_gpu_multiproc.py -q -p no:cacheprovider --timeout 900 > gpurun_out/r02ww_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02ww_multiproc.log
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621"
timeout 600 $RUN2 bench.py --gpus 2 > gpurun_out/r02ww_bench_n2.json 2> gpurun_out/r02ww_bench_n2.err
echo done
