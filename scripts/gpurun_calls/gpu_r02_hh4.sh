# 4 GPUs, one process: NVLink counters of rank 0's FUSED push to 1 and 3 peers (N=2 and N=4 shapes)
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for P in 1 3; do for s in threads bulk; do
  timeout 300 python scripts/nvl_redirect.py --scatter $s --peers $P >> gpurun_out/r02hh_redirect.jsonl 2>> gpurun_out/r02hh_redirect.err
  timeout 300 ncu --metrics $M -k regex:"k_scatter" --clock-control none --csv --log-file gpurun_out/r02hh_nvl_p${P}_$s.csv python scripts/nvl_redirect.py --scatter $s --peers $P --steps 2 --warmup 1 > gpurun_out/r02hh_ncu_p${P}_$s.log 2>&1
done; done
echo done
