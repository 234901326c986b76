# session-2 baseline check of the restored tree: full GPU suite, bench N=1, launch list, full ncu of emit+scatter
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2a_tests.log 2>&1; echo rc=$? >> gpurun_out/s2a_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s2a_bench_n1.json 2> gpurun_out/s2a_bench_n1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2a_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2a_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2a_ncu_a.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:"k_emit_bulk|k_scatter|k_hist" -s 6 -c 3 -o gpurun_out/s2a_prof python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2a_ncu_b.log 2>&1
echo done
