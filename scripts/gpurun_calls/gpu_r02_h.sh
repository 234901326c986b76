# 1 GPU: warp-tile path v4 (table ranking, cursors, STG) -- parity (+debug bounds), R=8 sweep, bench, ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r02h_tests.log 2>&1; echo rc=$? >> gpurun_out/r02h_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02h_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02h_tests_debug.log
for B in 48 64 16 128 32 24; do python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02h_sweep_L8.jsonl 2>&1; done
python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 134217728 >> gpurun_out/r02h_sweep_L8.jsonl 2>&1
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02h_bench_n1.json 2> gpurun_out/r02h_bench_n1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w" -s 1 -c 1 -o gpurun_out/r02h_r8 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02h_ncu.log 2>&1
echo done
