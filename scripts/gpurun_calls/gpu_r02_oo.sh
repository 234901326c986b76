# 1 GPU: histogram occupancy variants (8 warps x 3 stages, 12 x 2, 16 x 1)
for v in main h12 h16; do
  if [ $v = main ]; then export RAFI_LIB_PATH=; else export RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so; fi
  echo "{\"variant\": \"$v\"}" >> gpurun_out/r02oo_sweep.jsonl
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 48 >> gpurun_out/r02oo_sweep.jsonl 2>&1
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 48 --L 1 --n 16777216 >> gpurun_out/r02oo_sweep.jsonl 2>&1
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 128 >> gpurun_out/r02oo_sweep.jsonl 2>&1
done
echo done
