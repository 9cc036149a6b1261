#!/bin/bash
# 4-GPU box: parity of the changed comm kernels at W = 4 / 2 (RS: peer-only stages,
# own chunk from registers; update: loads before the barrier; no per-thread
# membar.sys), comm microbench W = 4 (eager + CUDA graph), VGG-19 bs8 trace + lines.
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_comm.py tests/test_gpu_executor.py \
  -q -m gpu -x > gpurun_out/r02f_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02f_pytest.log
# ncu --set full on the real NVLink (W = 2 on GPUs 0,1; gloo only, barriers off)
for spec in "update:64:update_allgather_tma" "rs:64:reduce_scatter_tma" "oneshot:1:oneshot_update" "update:4:update_allgather_tma"; do
  IFS=: read kk mb kname <<< "$spec"
  CUDA_VISIBLE_DEVICES=0,1 timeout 300 $T --nproc-per-node 2 --master-port $((29640 + RANDOM % 50)) --no-python \
    tools/gpu/ncu_full_rank0.sh gpurun_out/r02f_full_${kk}_${mb}mb_n2 $kname \
    python tools/comm_profile.py --kernel $kk --mb $mb > gpurun_out/r02f_full_${kk}_${mb}mb_n2.log 2>&1
  echo "ncu full $kk ${mb}MB rc=$?"; tail -2 gpurun_out/r02f_full_${kk}_${mb}mb_n2.log
done
timeout 600 $T --nproc-per-node 4 --master-port 29631 tools/comm_bench.py --sizes-mb 0.25,1,4,16,64,256 \
  --check --phases > gpurun_out/r02f_comm_n4.jsonl 2> gpurun_out/r02f_comm_n4.err
echo "comm n4 eager rc=$?"
timeout 600 $T --nproc-per-node 4 --master-port 29632 tools/comm_bench.py --sizes-mb 0.25,1,4,16,64,256 \
  --graph > gpurun_out/r02f_comm_n4_graph.jsonl 2> gpurun_out/r02f_comm_n4_graph.err
echo "comm n4 graph rc=$?"
$R trace r02f_trace_vgg19_b8_n4 4 --model vgg19 --batch 8
python tools/trace_summary.py gpurun_out/r02f_trace_vgg19_b8_n4 --rank 0 > gpurun_out/r02f_trace_vgg19_b8_n4_summary.txt 2>&1
head -40 gpurun_out/r02f_trace_vgg19_b8_n4_summary.txt
$R bench r02f_vgg19_b8_n4 4 --model vgg19 --batch 8 --no-cpu-baseline
$R bench r02f_r101_n4 4 --no-cpu-baseline
$R bench r02f_r101_n2 2 --no-cpu-baseline
for M in "resnet101" "vgg19 --batch 8"; do
  tag=$(echo $M | tr -d ' -')
  $R bench r02f_ddp_${tag}_n4 4 --impl ddp --model $M
  $R bench r02f_ddpgraph_${tag}_n4 4 --impl ddp --ddp-graphs --model $M
done
