# 4 GPUs: final tree -- every GPU test (single + multi-GPU), debug parity, smoke, bench N=1/2/4 and the reference arm
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612"
timeout 3000 python -m pytest tests -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02final2_tests_4gpu.log 2>&1; echo rc=$? >> gpurun_out/r02final2_tests_4gpu.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -p no:cacheprovider --timeout 300 > gpurun_out/r02final2_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02final2_tests_debug.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02final2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02final2_smoke.log
timeout 600 python bench.py > gpurun_out/r02final2_bench_n1.json 2> gpurun_out/r02final2_bench_n1.err
timeout 600 $RUN2 bench.py --gpus 2 > gpurun_out/r02final2_bench_n2.json 2> gpurun_out/r02final2_bench_n2.err
timeout 600 $RUN4 bench.py --gpus 4 > gpurun_out/r02final2_bench_n4.json 2> gpurun_out/r02final2_bench_n4.err
timeout 300 python bench.py --impl reference > gpurun_out/r02final2_ref_n1.json 2> gpurun_out/r02final2_ref_n1.err
echo done
