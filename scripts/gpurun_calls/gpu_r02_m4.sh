# 4 GPUs: the configs[1] headline (8 ranks; 8/N logical ranks per GPU) at N=1/2/4, reference arm, ncu launch list + full capture of the N=1 scatter
RUN2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
RUN4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532"
python bench.py > gpurun_out/r02m_bench_n1.json 2> gpurun_out/r02m_bench_n1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02m_ref_n1.json 2> gpurun_out/r02m_ref_n1.err
$RUN2 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r02m_bench_n2.json 2> gpurun_out/r02m_bench_n2.err
$RUN4 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r02m_bench_n4.json 2> gpurun_out/r02m_bench_n4.err
$RUN4 bench.py --gpus 4 --no-cpu-baseline --no-e2e --scatter threads > gpurun_out/r02m_bench_n4_threads.json 2> gpurun_out/r02m_bench_n4_threads.err
$RUN2 bench.py --gpus 2 --no-cpu-baseline --no-e2e --scatter threads > gpurun_out/r02m_bench_n2_threads.json 2> gpurun_out/r02m_bench_n2_threads.err
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-extras"
python bench.py $A > gpurun_out/r02m_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_launches_n1.csv python bench.py $A > gpurun_out/r02m_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_w|k_hist_w|k_emit_bulk" -s 12 -c 3 -o gpurun_out/r02m_full_n1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-extras > gpurun_out/r02m_ncu_full.log 2>&1
echo done
