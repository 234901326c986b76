# 4 GPUs: NVLink ceilings, full multi-GPU parity (world 2 and 4), bench N=4/N=2 per scatter mode, cfg5 at N=4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 120 ./tools/p2p_bw > gpurun_out/s2j_p2p_n4.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 ./tools/p2p_bw > gpurun_out/s2j_p2p_n2.jsonl 2>&1
timeout 2400 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/s2j_mp.log 2>&1; echo rc=$? >> gpurun_out/s2j_mp.log
for m in auto threads; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29551 bench.py --gpus 4 --steps 10 --warmup 3 --scatter $m > gpurun_out/s2j_bench_n4_$m.json 2> gpurun_out/s2j_bench_n4_$m.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29552 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/s2j_bench_n2_auto.json 2> gpurun_out/s2j_bench_n2_auto.err
timeout 600 $TR --nproc-per-node 4 --master-port 29553 bench_suite.py cfg5 --gpus 4 > gpurun_out/s2j_cfg5_n4_auto.jsonl 2> gpurun_out/s2j_cfg5_n4_auto.err
echo done
