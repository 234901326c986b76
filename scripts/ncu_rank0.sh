#!/bin/bash
# torchrun --no-python wrapper: rank 0 runs under a single-pass ncu NVLink
# counter capture of the payload kernels (our scatter / copy kernels only --
# never the NCCL kernels, which wait on the peer); the other ranks run plain.
# usage: torchrun ... --no-python bash scripts/ncu_rank0.sh OUT.csv bench.py ARGS...
out=$1; shift
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum \
    -k regex:"k_scatter|k_copy" --clock-control none --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi
