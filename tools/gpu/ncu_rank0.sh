#!/bin/bash
# NVLink bytes per launch of multi-GPU kernels: ncu on rank 0 only, one pass of
# counters (no kernel replay -- a replayed launch would wait forever for peers
# that ran their copy once).  Other ranks run the same command unprofiled.
#   torchrun --no-python --nproc-per-node N tools/gpu/ncu_rank0.sh OUT.csv python tools/comm_bench.py ...
out=$1; shift
if [ "${LOCAL_RANK:-0}" = 0 ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
    --clock-control none --cache-control none --replay-mode kernel \
    -k "regex:${NCU_KERNELS:-reduce_scatter|update_allgather|oneshot|ce_reduce|nccl}" \
    --csv --log-file "$out" "$@"
else
  exec "$@"
fi
