# 1 GPU: ILP of the untracked 8/4-byte-unit loop (8 vs 16 units in flight per lane)
for v in main n16; do
  if [ $v = main ]; then export RAFI_LIB_PATH=; else export RAFI_LIB_PATH=paper_2605_30294_b200/_variants/librafi_$v.so; fi
  for B in 20 40 44; do echo "{\"variant\": \"$v\"}" >> gpurun_out/r02dd_sweep.jsonl; timeout 300 python scripts/prof_binning.py --tiles 0 --scatter threads --B $B >> gpurun_out/r02dd_sweep.jsonl 2>&1; done
done
echo done
