# 1 GPU: final N=1 bench, launch list and full ncu capture of emit/hist/scatter (round-1 evidence)
python bench.py --steps 10 --warmup 3 > gpurun_out/s3e_bench_n1.json 2> gpurun_out/s3e_bench_n1.err
timeout 120 ./tools/p2p_bw > gpurun_out/s3e_p2p_n1.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3e_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3e_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3e_ncu_a.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:"k_emit_bulk|k_scatter|k_hist" -s 6 -c 3 -o gpurun_out/s3e_prof python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3e_ncu_b.log 2>&1
echo done
