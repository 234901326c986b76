# 4 GPUs: NVLink ceilings (fixed a2a), parity at world 4, bench N=4/N=2, latency+cfg1 at N=4 peer vs nccl control
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 120 ./tools/p2p_bw > gpurun_out/s2w_p2p_n4.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 ./tools/p2p_bw > gpurun_out/s2w_p2p_n2.jsonl 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29571 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/s2w_bench_n4.json 2> gpurun_out/s2w_bench_n4.err
for ctl in peer nccl; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29572 bench_suite.py latency --gpus 4 --control $ctl > gpurun_out/s2w_lat_n4_$ctl.jsonl 2> gpurun_out/s2w_lat_n4_$ctl.err
  timeout 300 $TR --nproc-per-node 4 --master-port 29573 bench_suite.py cfg4 --gpus 4 --control $ctl > gpurun_out/s2w_cfg4_n4_$ctl.jsonl 2> gpurun_out/s2w_cfg4_n4_$ctl.err
done
RAFI_TEST_WORLDS=4 timeout 2400 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/s2w_mp.log 2>&1; echo rc=$? >> gpurun_out/s2w_mp.log
echo done
