# 2 GPUs: NVLink ceilings, multi-GPU parity (all scatter write paths), bench N=2 per scatter mode
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/s2h_topo.txt 2>&1
timeout 120 ./tools/p2p_bw > gpurun_out/s2h_p2p.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -x -q -k "not 4" > gpurun_out/s2h_mp.log 2>&1; echo rc=$? >> gpurun_out/s2h_mp.log
for m in threads bulk aligned; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --scatter $m --no-e2e > gpurun_out/s2h_bench_n2_$m.json 2> gpurun_out/s2h_bench_n2_$m.err
done
timeout 600 $TR --nproc-per-node 2 --master-port 29532 bench_suite.py cfg5 --gpus 2 --scatter aligned > gpurun_out/s2h_cfg5_n2_aligned.jsonl 2> gpurun_out/s2h_cfg5_n2_aligned.err
echo done
