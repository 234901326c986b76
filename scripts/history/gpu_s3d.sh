# 4 GPUs: full GPU suite (single + multi-GPU), benches N=1/2/4, suites at N=4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 10 --warmup 3 > gpurun_out/s3d_bench_n1.json 2> gpurun_out/s3d_bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/s3d_bench_n2.json 2> gpurun_out/s3d_bench_n2.err
timeout 300 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/s3d_bench_n4.json 2> gpurun_out/s3d_bench_n4.err
for w in cfg3 cfg4 cfg5 sweep nbody; do
  timeout 600 $TR --nproc-per-node 4 --master-port 29613 bench_suite.py $w --gpus 4 > gpurun_out/s3d_n4_$w.jsonl 2> gpurun_out/s3d_n4_$w.err
done
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/s3d_tests.log 2>&1; echo rc=$? >> gpurun_out/s3d_tests.log
echo done
