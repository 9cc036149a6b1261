#!/bin/bash
# 2-GPU box: update ring chunk 2048 vs 4096 elements -- loopback parity with 4096,
# W=2 comm microbench at the step's 32-CTA update budget, ResNet-101 N=2 lines.
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
DEFT_UPDATE_TMA_CHUNK=4096 timeout 400 python -m pytest tests/test_gpu_loopback.py -q -m gpu -x \
  -k "update_allgather or deft_fp32 or deft_bf16" > gpurun_out/r02h_pytest_chunk4096.log 2>&1
echo "pytest chunk4096 rc=$?"; tail -2 gpurun_out/r02h_pytest_chunk4096.log
for C in 2048 4096; do
  DEFT_UPDATE_TMA_CHUNK=$C timeout 300 $T --master-port $((29700 + C % 97)) tools/comm_bench.py \
    --sizes-mb 16,64 --update-blocks 32 --graph --no-nccl > gpurun_out/r02h_comm_n2_b32_c$C.jsonl 2> gpurun_out/r02h_comm_n2_b32_c$C.err
  echo "comm c$C rc=$?"
done
for C in 2048 4096; do
  DEFT_UPDATE_TMA_CHUNK=$C timeout 420 $T --master-port $((29750 + C % 89)) bench.py --gpus 2 --no-cpu-baseline \
    > gpurun_out/r02h_r101_n2_c$C.json 2> gpurun_out/r02h_r101_n2_c$C.err
  echo "bench c$C rc=$? $(tail -c 200 gpurun_out/r02h_r101_n2_c$C.json)"
done
