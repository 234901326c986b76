# 1 GPU: final single-GPU suite, smoke, bench, launch list and full ncu capture (round-1 final evidence)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3k_tests.log 2>&1; echo rc=$? >> gpurun_out/s3k_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3k_smoke.log 2>&1; echo rc=$? >> gpurun_out/s3k_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s3k_bench_n1.json 2> gpurun_out/s3k_bench_n1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3k_ref_n1.json 2> gpurun_out/s3k_ref_n1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3k_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3k_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3k_ncu_a.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:"k_emit_bulk|k_scatter|k_hist" -s 6 -c 3 -o gpurun_out/s3k_prof python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3k_ncu_b.log 2>&1
echo done
