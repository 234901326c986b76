# 2 GPUs: N=2 blocking-step diagnostic; single-process FUSED NVLink push (redirect) timed and under ncu NVLink counters
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k redirect > gpurun_out/r02j_tests.log 2>&1; echo rc=$? >> gpurun_out/r02j_tests.log
timeout 300 $RUN scripts/diag_n2.py > gpurun_out/r02j_diag_n2.jsonl 2> gpurun_out/r02j_diag_n2.err
for s in threads bulk; do timeout 300 python scripts/nvl_redirect.py --scatter $s >> gpurun_out/r02j_redirect.jsonl 2>> gpurun_out/r02j_redirect.err; done
M=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for s in threads bulk; do timeout 300 ncu --metrics $M -k regex:"k_scatter" --clock-control none --csv --log-file gpurun_out/r02j_nvl_ncu_$s.csv python scripts/nvl_redirect.py --scatter $s --steps 2 --warmup 1 > gpurun_out/r02j_nvl_ncu_$s.log 2>&1; done
timeout 300 ncu --metrics $M -k regex:"k_copy16|k_push|k_" -c 6 --clock-control none --csv --log-file gpurun_out/r02j_p2p_ncu.csv tools/p2p_bw > gpurun_out/r02j_p2p_ncu.log 2>&1
echo done
