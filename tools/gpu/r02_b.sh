#!/bin/bash
# 4-GPU box: comm microbench (one-shot / two-shot / NCCL, NVML NVLink bytes) at
# W = 4 and 2; W = 1 update variants on GPU 0; VGG-19 bs8 N=4 deferral policies;
# default ResNet-101 N=4 / N=2 lines.
mkdir -p gpurun_out
run() { # N tag args...
  local N=$1 tag=$2; shift 2
  if [ "$N" = 1 ]; then timeout 900 python bench.py "$@" > gpurun_out/$tag.json 2> gpurun_out/$tag.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $N "$@" > gpurun_out/$tag.json 2> gpurun_out/$tag.err; fi
  echo "$tag rc=$? $(head -c 400 gpurun_out/$tag.json)"
}
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_executor.py -q -m gpu \
  -k "deferral or not loopback" > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02b_pytest.log
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29517 tools/comm_bench.py \
    --sizes-mb 0.25,1,4,16,64,256 --nvml --check > gpurun_out/r02_comm_n$N.jsonl 2> gpurun_out/r02_comm_n$N.err
  echo "comm n=$N rc=$?"; tail -2 gpurun_out/r02_comm_n$N.err
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/update_bench.py > gpurun_out/r02_update_w1.jsonl 2>&1
echo "update_bench rc=$?"; cat gpurun_out/r02_update_w1.jsonl
run 4 r02_vgg19_b8_n4_last --model vgg19 --batch 8 --no-cpu-baseline --defer last
run 4 r02_vgg19_b8_n4_pred --model vgg19 --batch 8 --no-cpu-baseline --defer predicted
run 4 r02_vgg19_b8_n4_none --model vgg19 --batch 8 --no-cpu-baseline --defer none
run 4 r02_r101_n4 --no-cpu-baseline
run 2 r02_r101_n2 --no-cpu-baseline
