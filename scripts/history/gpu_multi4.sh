set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/mp4.log 2>&1; echo rc=$? >> gpurun_out/mp4.log
timeout 300 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b4_n4.json 2> gpurun_out/b4_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b4_n2.json 2> gpurun_out/b4_n2.err
for w in cfg4 cfg3 cfg5 sweep; do timeout 600 $TR --nproc-per-node 4 --master-port 29513 bench_suite.py $w --gpus 4 > gpurun_out/s4_n4_$w.jsonl 2> gpurun_out/s4_n4_$w.err; done
for w in cfg4 cfg3 latency cfg1; do CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29514 bench_suite.py $w --gpus 2 > gpurun_out/s4_n2_$w.jsonl 2> gpurun_out/s4_n2_$w.err; done
