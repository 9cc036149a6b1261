#!/bin/bash
# 4-GPU box: update ring chunk 4096 vs 2048 in the comm-heavy step (VGG-19 bs8) and ResNet-101.
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for spec in "4096:vgg19 --batch 8" "2048:vgg19 --batch 8" "4096:resnet101"; do
  C=${spec%%:*} M=${spec#*:}; tag=$(echo $M | tr -d ' -')
  DEFT_UPDATE_TMA_CHUNK=$C timeout 300 $T --master-port $((29800 + RANDOM % 90)) bench.py --gpus 4 \
    --no-cpu-baseline --model $M > gpurun_out/r02i_${tag}_n4_c$C.json 2> gpurun_out/r02i_${tag}_n4_c$C.err
  echo "$tag c$C rc=$? $(tail -c 150 gpurun_out/r02i_${tag}_n4_c$C.json)"
done
