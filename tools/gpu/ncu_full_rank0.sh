#!/bin/bash
# ncu --set full of ONE multi-GPU comm kernel launch, on rank 0, with kernel
# replay: DEFT_PROFILE_NO_PEER_BARRIER=1 turns the cross-GPU barriers off on
# every rank (racy results -- profiling only), so each replayed pass streams
# over the real NVLink without waiting for peers that ran their copy once.
#   torchrun --no-python --nproc-per-node N tools/gpu/ncu_full_rank0.sh OUT KERNEL_REGEX \
#       python tools/comm_bench.py --no-nccl --sizes-mb 64 --reps 3
out=$1 k=$2; shift 2
export DEFT_PROFILE_NO_PEER_BARRIER=1
if [ "${LOCAL_RANK:-0}" = 0 ]; then
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s ${NCU_SKIP:-2} -c 1 \
    -o "$out" "$@"
  rc=$?
  ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>&1
  exit $rc
else
  exec "$@"
fi
