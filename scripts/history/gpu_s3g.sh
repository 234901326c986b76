# 2 GPUs: final suite numbers at N=1 and N=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for w in sweep cfg1 cfg3 cfg4 nbody streamlines latency; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_suite.py $w > gpurun_out/s3g_n1_$w.jsonl 2> gpurun_out/s3g_n1_$w.err
done
for w in sweep cfg1 cfg3 cfg4 latency; do
  timeout 600 $TR --nproc-per-node 2 --master-port 29621 bench_suite.py $w --gpus 2 > gpurun_out/s3g_n2_$w.jsonl 2> gpurun_out/s3g_n2_$w.err
done
echo done
