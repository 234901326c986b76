# 1 GPU: warp scatter with one TMA stage per warp (up to 16 warps/SM) vs two
for rep in 1 2; do for v in main w1; do
  if [ $v = main ]; then export RAFI_LIB_PATH=; else export RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so; fi
  echo "{\"variant\": \"$v\"}" >> gpurun_out/r02rr_sweep.jsonl
  for B in 16 44 48 64 128; do timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02rr_sweep.jsonl 2>&1; done
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --L 1 --n 16777216 >> gpurun_out/r02rr_sweep.jsonl 2>&1
done; done
echo done
