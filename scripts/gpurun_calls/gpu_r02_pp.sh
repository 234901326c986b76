# 1 GPU: histogram warps x stages variants, repeated
for rep in 1 2; do for v in main h16 h16b h12; do
  if [ $v = main ]; then export RAFI_LIB_PATH=; else export RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so; fi
  echo "{\"variant\": \"$v\"}" >> gpurun_out/r02pp_sweep.jsonl
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 48 >> gpurun_out/r02pp_sweep.jsonl 2>&1
  timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B 128 >> gpurun_out/r02pp_sweep.jsonl 2>&1
done; done
echo done
