# 2 GPUs, same box: peer vs nccl control on latency-bound rounds (latency, cfg1, sweep small sizes)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2; do for ctl in peer nccl; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29581 bench_suite.py latency --gpus 2 --control $ctl > gpurun_out/s2y_lat_${ctl}_$rep.jsonl 2>/dev/null
  timeout 300 $TR --nproc-per-node 2 --master-port 29582 bench_suite.py cfg1 --gpus 2 --control $ctl > gpurun_out/s2y_cfg1_${ctl}_$rep.jsonl 2>/dev/null
done; done
for ctl in peer nccl; do
  timeout 600 $TR --nproc-per-node 2 --master-port 29583 bench_suite.py sweep --gpus 2 --control $ctl > gpurun_out/s2y_sweep_$ctl.jsonl 2>/dev/null
done
timeout 300 $TR --nproc-per-node 2 --master-port 29584 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/s2y_bench_n2.json 2> gpurun_out/s2y_bench_n2.err
echo done
