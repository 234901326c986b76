# 2 GPUs: parity (world 2) with scan/scatter-fused peer control; A/B latency, cfg1, sweep; bench N=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
RAFI_TEST_WORLDS=2 timeout 1500 python -m pytest tests/test_gpu_multiproc.py -x -q -k "control or hybrid or (snapshot and 48)" > gpurun_out/s2z_mp.log 2>&1; echo rc=$? >> gpurun_out/s2z_mp.log
for rep in 1 2; do for ctl in peer nccl; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29591 bench_suite.py latency --gpus 2 --control $ctl > gpurun_out/s2z_lat_${ctl}_$rep.jsonl 2>/dev/null
  timeout 300 $TR --nproc-per-node 2 --master-port 29592 bench_suite.py cfg1 --gpus 2 --control $ctl > gpurun_out/s2z_cfg1_${ctl}_$rep.jsonl 2>/dev/null
done; done
for ctl in peer nccl; do
  timeout 600 $TR --nproc-per-node 2 --master-port 29593 bench_suite.py sweep --gpus 2 --control $ctl > gpurun_out/s2z_sweep_$ctl.jsonl 2>/dev/null
  timeout 300 $TR --nproc-per-node 2 --master-port 29594 bench.py --gpus 2 --steps 10 --warmup 3 --control $ctl --no-e2e > gpurun_out/s2z_bench_n2_$ctl.json 2>/dev/null
done
echo done
