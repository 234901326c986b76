# 1 GPU: shared-device tests, bench (with binning_r8 / device_emit), launch list, full ncu of the hot kernels
timeout 900 python -m pytest tests/test_gpu_shared_device.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "shared or two_processes or overflow or reemit" > gpurun_out/r02c_tests.log 2>&1; echo rc=$? >> gpurun_out/r02c_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02c_bench_n1.json 2> gpurun_out/r02c_bench_n1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02c_ref_n1.json 2> gpurun_out/r02c_ref_n1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02c_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02c_ncu_a.log 2>&1
echo done
