# 4 GPUs: the suite at N=2 and N=4 on the round-2 kernels (8-rank configs: 8/N logical ranks per GPU); multi-GPU parity
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552"
for w in cfg5 cfg3 cfg4 nbody streamlines cfg1 latency sweep; do timeout 900 $RUN4 bench_suite.py $w --gpus 4 > gpurun_out/r02z_suite_n4_$w.jsonl 2> gpurun_out/r02z_suite_n4_$w.err; done
for w in cfg5 sweep; do timeout 900 $RUN2 bench_suite.py $w --gpus 2 > gpurun_out/r02z_suite_n2_$w.jsonl 2> gpurun_out/r02z_suite_n2_$w.err; done
timeout 2400 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider --timeout 900 > gpurun_out/r02z_multiproc.log 2>&1; echo rc=$? >> gpurun_out/r02z_multiproc.log
echo done
