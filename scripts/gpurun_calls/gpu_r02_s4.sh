# 4 GPUs: final-tree validation -- multi-GPU parity (world 2 and 4), bench configs[1] at N=1/2/4, reference arm
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542"
timeout 600 python bench.py > gpurun_out/r02s_bench_n1.json 2> gpurun_out/r02s_bench_n1.err
timeout 600 $RUN2 bench.py --gpus 2 > gpurun_out/r02s_bench_n2.json 2> gpurun_out/r02s_bench_n2.err
timeout 600 $RUN4 bench.py --gpus 4 > gpurun_out/r02s_bench_n4.json 2> gpurun_out/r02s_bench_n4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02s_ref_n1.json 2> gpurun_out/r02s_ref_n1.err
timeout 300 $RUN4 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/r02s_ref_n4.json 2> gpurun_out/r02s_ref_n4.err
timeout 2400 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider --timeout 900 > gpurun_out/r02s_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02s_multiproc.log
echo done
