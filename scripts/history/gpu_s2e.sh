# ncu of the bulk scatter, 48 B, tile 256 (2 output buffers, 4 CTAs/SM) vs tile 512 (1 buffer, 2 CTAs/SM)
for T in 256 512; do
python bench_suite.py cfg5 --scatter bulk --tile $T --sizes 48 --items 8388608 > gpurun_out/s2e_plain_$T.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_scatter_bulk" -s 3 -c 1 -o gpurun_out/s2e_bulk_T$T python bench_suite.py cfg5 --scatter bulk --tile $T --sizes 48 --items 8388608 > gpurun_out/s2e_ncu_$T.log 2>&1
done
echo done
