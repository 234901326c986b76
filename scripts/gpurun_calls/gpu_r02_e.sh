# 1 GPU: warp-tile binning path -- parity, R=8/R=1 sweeps vs block tiles, bench, ncu of the warp scatter
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1; echo rc=$? >> gpurun_out/r02e_tests.log
for B in 48 64 16 128 24; do python scripts/prof_binning.py --tiles 0,512,2048 --scatter threads --B $B >> gpurun_out/r02e_sweep_L8.jsonl 2>&1; done
python scripts/prof_binning.py --tiles 0,512,2048 --scatter threads --L 1 --n 134217728 > gpurun_out/r02e_sweep_L1.jsonl 2>&1
python scripts/prof_binning.py --tiles 0,512 --scatter threads --L 1 --n 16777216 > gpurun_out/r02e_sweep_L1_16M.jsonl 2>&1
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02e_bench_n1.json 2> gpurun_out/r02e_bench_n1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w|k_hist_w" -s 2 -c 2 -o gpurun_out/r02e_r8 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02e_ncu.log 2>&1
echo done
