TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 10 --warmup 3 > gpurun_out/bench14_n1.json 2> gpurun_out/bench14_n1.err
timeout 300 $TR --nproc-per-node 2 --master-port 29515 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench14_n2.json 2> gpurun_out/bench14_n2.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_suite.py sweep > gpurun_out/sweep14.jsonl 2>&1
