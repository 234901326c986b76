# 1 GPU: ncu --set full of the warp-tile histogram (R=8, 8 x 16M)
timeout 300 python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02nn_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hist_w" -s 1 -c 1 -o gpurun_out/r02nn_hist python scripts/prof_binning.py --tiles 0 --steps 1 --warmup 1 > gpurun_out/r02nn_ncu.log 2>&1
echo done
