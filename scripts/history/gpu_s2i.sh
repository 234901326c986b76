# 2 GPUs: full multi-GPU parity at world 2 (all exchanges incl. CE, all scatter write paths), bench N=2 CE vs FUSED
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
RAFI_TEST_WORLDS=2 timeout 1500 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/s2i_mp.log 2>&1; echo rc=$? >> gpurun_out/s2i_mp.log
for ex in ce fused; do for m in threads bulk; do
  timeout 300 $TR --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 --exchange $ex --scatter $m --no-e2e > gpurun_out/s2i_bench_n2_${ex}_$m.json 2> gpurun_out/s2i_bench_n2_${ex}_$m.err
done; done
echo done
