# 1 GPU: warp-tile path v2 (prefetched run bases, persistent TMA hist)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r02f_tests.log 2>&1; echo rc=$? >> gpurun_out/r02f_tests.log
for B in 48 64 16 128 24 32; do python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02f_sweep_L8.jsonl 2>&1; done
python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 134217728 > gpurun_out/r02f_sweep_L1.jsonl 2>&1
python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 16777216 > gpurun_out/r02f_sweep_L1_16M.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w|k_hist_w" -s 2 -c 2 -o gpurun_out/r02f_r8 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02f_ncu.log 2>&1
echo done
