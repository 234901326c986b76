# 1 GPU: fused count kernel (hist + look-back scan) -- parity (+debug bounds), graph, shared-device, bench, R=8/R=1 timings, ncu launch list
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py tests/test_gpu_shared_device.py tests/test_gpu_protocol.py -x -q -p no:cacheprovider > gpurun_out/r02l_tests.log 2>&1; echo rc=$? >> gpurun_out/r02l_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > gpurun_out/r02l_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02l_tests_debug.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02l_bench_n1.json 2> gpurun_out/r02l_bench_n1.err
for B in 48 64 32; do python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02l_sweep.jsonl 2>&1; done
python scripts/prof_binning.py --tiles 0,512,0,512 --scatter threads --L 1 --n 16777216 >> gpurun_out/r02l_sweep.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02l_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02l_ncu_launch.log 2>&1
echo done
