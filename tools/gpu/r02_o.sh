#!/bin/bash
# 2-GPU box: final-kernel W=2 comm sweep (CUDA-graph timing) vs NCCL.
mkdir -p gpurun_out
timeout 400 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 \
  --master-port 29931 tools/comm_bench.py --sizes-mb 1,4,16,64,256 --graph \
  > gpurun_out/r02o_comm_n2_graph.jsonl 2> gpurun_out/r02o_comm_n2_graph.err
echo "comm rc=$?"
