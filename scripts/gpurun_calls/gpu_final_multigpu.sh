# 4 GPUs: multi-GPU parity with the graph-replayed forward (world 2 and 4), benches N=2/N=4, suites at N=4 and N=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29631 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/s3j_bench_n2.json 2> gpurun_out/s3j_bench_n2.err
timeout 300 $TR --nproc-per-node 4 --master-port 29632 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/s3j_bench_n4.json 2> gpurun_out/s3j_bench_n4.err
for w in sweep cfg4 cfg3 cfg5; do
  timeout 600 $TR --nproc-per-node 4 --master-port 29633 bench_suite.py $w --gpus 4 > gpurun_out/s3j_n4_$w.jsonl 2> gpurun_out/s3j_n4_$w.err
done
for w in sweep cfg1 latency cfg4; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29634 bench_suite.py $w --gpus 2 > gpurun_out/s3j_n2_$w.jsonl 2> gpurun_out/s3j_n2_$w.err
done
timeout 3000 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/s3j_mp.log 2>&1; echo rc=$? >> gpurun_out/s3j_mp.log
echo done
