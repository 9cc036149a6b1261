#!/bin/bash
# Round-2 validation on a 4-GPU box: GPU tests (incl. multigpu), smoke, then the
# comm microbench (one-shot vs two-shot vs NCCL, NVML NVLink bytes) at W=2 and 4.
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r02_topo.txt 2>&1
tools/gpu/validate.sh r02a
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29517 tools/comm_bench.py \
    --sizes-mb 0.25,1,4,16,64,256 --nvml --check > gpurun_out/r02_comm_n$N.jsonl 2> gpurun_out/r02_comm_n$N.err
  echo "comm n=$N rc=$?"; tail -3 gpurun_out/r02_comm_n$N.err
done
