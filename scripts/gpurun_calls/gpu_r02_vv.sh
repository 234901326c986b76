# 1 GPU: two stages up to 96 B -- full GPU suite (+debug parity), 96/128-B sweep, bench
timeout 1800 python -m pytest tests -q -p no:cacheprovider -m gpu --timeout 900 > gpurun_out/r02vv_tests.log 2>&1; echo rc=$? >> gpurun_out/r02vv_tests.log
RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -p no:cacheprovider --timeout 300 > gpurun_out/r02vv_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/r02vv_tests_debug.log
for B in 96 128 48; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02vv_sweep.jsonl 2>&1; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02vv_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02vv_smoke.log
timeout 600 python bench.py > gpurun_out/r02vv_bench_n1.json 2> gpurun_out/r02vv_bench_n1.err
echo done
