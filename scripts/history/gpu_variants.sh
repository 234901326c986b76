# scatter tuning variants (build.py --variants): cfg5 item-size sweep at 16M items/rank, 1 GPU
timeout 300 python bench_suite.py cfg5 --items 16777216 > gpurun_out/var_default.jsonl 2>&1
for v in minb3 minb4 ilp8 minb3_ilp8; do
  RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so timeout 300 python bench_suite.py cfg5 --items 16777216 > gpurun_out/var_$v.jsonl 2>&1
done
