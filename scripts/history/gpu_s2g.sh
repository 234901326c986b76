# ncu: threads vs aligned scatter at 16 B and 44 B (8M items, R=1)
for m in threads aligned; do for B in ${SIZES:-16}; do
python bench_suite.py cfg5 --scatter $m --sizes $B --items 8388608 > gpurun_out/s2g_plain_${m}_$B.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 3 -c 1 -o gpurun_out/s2g_${m}_$B python bench_suite.py cfg5 --scatter $m --sizes $B --items 8388608 > gpurun_out/s2g_ncu_${m}_$B.log 2>&1
done; done
echo done
