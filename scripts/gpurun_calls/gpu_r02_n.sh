# 1 GPU: 128/256-item warp tiles -- parity (+debug), tile sweep per item size, bench N=1, full ncu of the bench's scatter
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/r02n_tests.log 2>&1; echo rc=$? >> gpurun_out/r02n_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tile or warp_tiles or redirect" --timeout 300 > gpurun_out/r02n_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02n_tests_debug.log
for B in 16 24 32 48 56 64 96 128; do timeout 300 python scripts/prof_binning.py --tiles 128,256 --scatter threads --B $B >> gpurun_out/r02n_sweep.jsonl 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02n_bench_n1.json 2> gpurun_out/r02n_bench_n1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w" -s 1 -c 1 -o gpurun_out/r02n_full_scatter python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02n_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_emit_bulk|k_hist_w" -s 18 -c 2 -o gpurun_out/r02n_full_emit_hist python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02n_ncu_full2.log 2>&1
echo done
