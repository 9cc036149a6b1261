#!/bin/bash
# 2-GPU box: parity of the changed update kernel (loads before the entry barrier,
# no per-thread membar.sys); where the fixed per-launch cost of the comm kernels
# goes (phase stamps, barrier fence A/B); ncu --set full of the update /
# reduce-scatter / one-shot kernels on the real NVLink (rank 0, peer barriers off).
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 1200 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_comm.py tests/test_gpu_executor.py \
  -q -m gpu -x > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02e_pytest.log
timeout 600 $T --master-port 29611 tools/comm_bench.py --sizes-mb 0.25,1,4,16,64 --phases --reps 20 \
  > gpurun_out/r02e_phases_n2.jsonl 2> gpurun_out/r02e_phases_n2.err
echo "phases rc=$?"
DEFT_BARRIER_FENCE=all timeout 600 $T --master-port 29612 tools/comm_bench.py --sizes-mb 0.25,1,4,16,64 \
  --phases --reps 20 > gpurun_out/r02e_phases_n2_fenceall.jsonl 2> gpurun_out/r02e_phases_n2_fenceall.err
echo "phases fence=all rc=$?"
for spec in "update_allgather_tma:64" "reduce_scatter_tma:64" "oneshot_update:1" "update_allgather_tma:4"; do
  k=${spec%%:*} mb=${spec##*:}
  timeout 600 $T --master-port $((29620 + RANDOM % 50)) --no-python tools/gpu/ncu_full_rank0.sh \
    gpurun_out/r02e_full_${k}_${mb}mb_n2 $k python tools/comm_bench.py --sizes-mb $mb --reps 3 --no-nccl \
    > gpurun_out/r02e_full_${k}_${mb}mb_n2.log 2>&1
  echo "ncu full $k ${mb}MB rc=$?"; tail -2 gpurun_out/r02e_full_${k}_${mb}mb_n2.log
done
