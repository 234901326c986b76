# 4 GPUs: bulk-scatter tile sweep for NVLink pushes (N=4 and N=2)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for T in 256 512 1024; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29601 bench_suite.py cfg5 --gpus 4 --scatter bulk --tile $T --sizes 44,48,64 --items 16777216 > gpurun_out/s3c_n4_T$T.jsonl 2>/dev/null
  CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29602 bench_suite.py cfg5 --gpus 2 --scatter bulk --tile $T --sizes 44,48,64 --items 16777216 > gpurun_out/s3c_n2_T$T.jsonl 2>/dev/null
done
echo done
