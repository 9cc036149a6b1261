#!/bin/bash
# 4-GPU box: update-kernel store pipelining (DEFT_UPDATE_TMA_PIPE) -- parity, comm
# microbench at W = 2 / 4 with NVML NVLink byte counters, in-step ResNet-101 N = 2;
# W = 1 sgd_local grid; default N = 1 line.
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
timeout 1200 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_comm.py -q -m gpu -x \
  -k "deft_fp32 or deft_bf16 or oneshot or multi_gpu or reduce_scatter" > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02c_pytest.log
$R comm 4 1,4,16,64,256; mv gpurun_out/comm_n4.jsonl gpurun_out/r02c_comm_n4.jsonl; cp gpurun_out/comm_n4.err gpurun_out/r02c_comm_n4.err
for PIPE in 3:0 4:1 6:2; do
  DEFT_UPDATE_TMA_PIPE=$PIPE $R comm 2 4,16,64,256
  mv gpurun_out/comm_n2.jsonl gpurun_out/r02c_comm_n2_pipe${PIPE/:/}.jsonl
done
$R update_w1 --grid 2:16,2:32,4:16,1:16; mv gpurun_out/update_w1.jsonl gpurun_out/r02c_update_w1.jsonl
for PIPE in 3:0 4:1 6:2; do
  DEFT_UPDATE_TMA_PIPE=$PIPE $R bench r02c_r101_n2_pipe${PIPE/:/} 2 --no-cpu-baseline
done
$R bench r02c_r101_n4 4 --no-cpu-baseline
$R bench r02c_r101_n1 1
