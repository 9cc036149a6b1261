#!/bin/bash
# 2-GPU box: bench lines with the isolated kernels timed cold per pass (L2 flushed) + CUDA graph.
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/r02l_r101_n1.json 2> gpurun_out/r02l_r101_n1.err
echo "bench n1 rc=$? $(tail -c 150 gpurun_out/r02l_r101_n1.json)"
timeout 400 $T --master-port 29881 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r02l_r101_n2.json 2> gpurun_out/r02l_r101_n2.err
echo "bench n2 rc=$? $(tail -c 150 gpurun_out/r02l_r101_n2.json)"
