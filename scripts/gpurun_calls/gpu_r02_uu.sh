# 1 GPU: final-tree ncu evidence of the bench -- launch list and --set full of the dominant scatter and the histogram
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras"
python bench.py $A > gpurun_out/r02uu_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02uu_launches_n1.csv python bench.py $A > gpurun_out/r02uu_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w|k_hist_w" -s 2 -c 2 -o gpurun_out/r02uu_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02uu_ncu_full.log 2>&1
echo done
