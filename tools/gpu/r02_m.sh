#!/bin/bash
# 4-GPU box: copy-engine channel with the W-1 peer pulls on parallel streams --
# loopback + multi-GPU CE parity, then VGG-19 bs8 N=4 parallel vs serial pulls.
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 420 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_comm.py -q -m gpu -x \
  -k "reduce_scatter or deft_fp32 or deft_bf16 or multi_gpu" > gpurun_out/r02m_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02m_pytest.log
for P in 1 0; do
  DEFT_CE_PARALLEL=$P timeout 240 $T --master-port $((29900 + P)) bench.py --gpus 4 --no-cpu-baseline \
    --model vgg19 --batch 8 > gpurun_out/r02m_vgg19_b8_n4_cepar$P.json 2> gpurun_out/r02m_vgg19_b8_n4_cepar$P.err
  echo "vgg cepar$P rc=$? $(tail -c 120 gpurun_out/r02m_vgg19_b8_n4_cepar$P.json)"
done
