# 1 GPU: emit tests, R=8 tile sweeps (threads/bulk, 48 B and 64 B), device-emit bench, ncu of the R=8 scatter
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared_device.py -q -p no:cacheprovider -k "reemit or overflow or two_processes" > gpurun_out/r02d_tests.log 2>&1; echo rc=$? >> gpurun_out/r02d_tests.log
python scripts/prof_binning.py --tiles 256,512,1024,2048,4096 --scatter threads > gpurun_out/r02d_sweep_threads48.jsonl 2>&1
python scripts/prof_binning.py --tiles 256,512,1024,2048 --scatter bulk > gpurun_out/r02d_sweep_bulk48.jsonl 2>&1
python scripts/prof_binning.py --tiles 256,512,1024,2048 --scatter threads --L 1 --n 134217728 > gpurun_out/r02d_sweep_threads48_L1.jsonl 2>&1
python scripts/prof_binning.py --tiles 256,512,1024,2048 --scatter threads --B 64 > gpurun_out/r02d_sweep_threads64.jsonl 2>&1
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02d_bench_n1.json 2> gpurun_out/r02d_bench_n1.err
python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02d_prof_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_hist" -s 2 -c 2 -o gpurun_out/r02d_r8 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02d_ncu.log 2>&1
echo done
