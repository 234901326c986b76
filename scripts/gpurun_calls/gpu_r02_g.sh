# 1 GPU: warp-tile path v3 (deferred run-base adds) + stage/unroll variants + debug-bounds parity
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1; echo rc=$? >> gpurun_out/r02g_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02g_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02g_tests_debug.log
for v in main w3 u4; do
  if [ $v = main ]; then export RAFI_LIB_PATH=; else export RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so; fi
  for B in 48 64 16 128 32; do echo "{\"variant\": \"$v\"}" >> gpurun_out/r02g_sweep_L8.jsonl; python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02g_sweep_L8.jsonl 2>&1; done
  python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 134217728 >> gpurun_out/r02g_sweep_L8.jsonl 2>&1
done
unset RAFI_LIB_PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w" -s 1 -c 1 -o gpurun_out/r02g_r8 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02g_ncu.log 2>&1
echo done
