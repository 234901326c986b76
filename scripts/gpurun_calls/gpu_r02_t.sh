# 1 GPU: ncu of the R=8 warp scatter at 44 B (chunk gather), 20 B (4-B units), 40 B (8-B units)
for B in 44 20 40; do timeout 300 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 --B $B > gpurun_out/r02t_plain_$B.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w" -s 1 -c 1 -o gpurun_out/r02t_b$B python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 --B $B > gpurun_out/r02t_ncu_$B.log 2>&1; done
echo done
