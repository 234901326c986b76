# 4 GPUs: multi-GPU parity (world 2 and 4) with the file rendezvous; bench N=4
timeout 2400 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider --timeout 900 > gpurun_out/r02ii_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02ii_multiproc.log
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581"
timeout 600 $RUN4 bench.py --gpus 4 > gpurun_out/r02ii_bench_n4.json 2> gpurun_out/r02ii_bench_n4.err
echo done
