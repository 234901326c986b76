# 2 GPUs: multi-GPU parity at world 2 (peer control default), bench N=2 nccl vs peer control
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
RAFI_TEST_WORLDS=2 timeout 1800 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/s2v_mp.log 2>&1; echo rc=$? >> gpurun_out/s2v_mp.log
for ctl in peer nccl; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29561 bench.py --gpus 2 --steps 10 --warmup 3 --control $ctl --no-e2e > gpurun_out/s2v_bench_n2_$ctl.json 2> gpurun_out/s2v_bench_n2_$ctl.err
done
timeout 300 $TR --nproc-per-node 2 --master-port 29562 bench_suite.py latency --gpus 2 > gpurun_out/s2v_lat_n2.jsonl 2> gpurun_out/s2v_lat_n2.err
timeout 300 $TR --nproc-per-node 2 --master-port 29563 bench_suite.py cfg1 --gpus 2 > gpurun_out/s2v_cfg1_n2.jsonl 2> gpurun_out/s2v_cfg1_n2.err
echo done
