# 2 GPUs: multi-GPU parity incl. bulk scatter to NVLink peers; bench N=2 threads vs bulk; cfg5 sweep N=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "not 4" > gpurun_out/s2c_mp.log 2>&1; echo rc=$? >> gpurun_out/s2c_mp.log
for m in threads bulk; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 10 --warmup 3 --scatter $m --no-e2e > gpurun_out/s2c_bench_n2_$m.json 2> gpurun_out/s2c_bench_n2_$m.err
  timeout 600 $TR --nproc-per-node 2 --master-port 29522 bench_suite.py cfg5 --gpus 2 --scatter $m > gpurun_out/s2c_cfg5_n2_$m.jsonl 2> gpurun_out/s2c_cfg5_n2_$m.err
done
echo done
