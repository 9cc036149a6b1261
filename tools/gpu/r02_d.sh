#!/bin/bash
# 4-GPU box: (1) N=1 A/B against the round-1 tree (_ab/r01, same box, alternating);
# (2) NVLink bytes per launch (ncu on rank 0, single pass) at W=4, 64 and 4 MB;
# (3) comm microbench W=4 (one-shot vs two-shot vs NCCL); (4) VGG-19 bs8 N=4.
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
for i in 1 2; do
  (cd _ab/r01 && timeout 600 python bench.py --no-cpu-baseline > ../../gpurun_out/r02d_ab_r01_$i.json 2> ../../gpurun_out/r02d_ab_r01_$i.err; echo "r01 tree rc=$? $(tail -c 200 ../../gpurun_out/r02d_ab_r01_$i.json)")
  $R bench r02d_ab_head_$i 1 --no-cpu-baseline
done
for MB in 64 4; do
  DEFT_SPIN_TIMEOUT_MS=30000 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29541 --no-python tools/gpu/ncu_rank0.sh \
    gpurun_out/r02d_nvl_n4_${MB}mb.csv python tools/comm_bench.py --sizes-mb $MB --reps 3 \
    > gpurun_out/r02d_nvl_n4_${MB}mb.log 2>&1
  echo "ncu nvlink ${MB}MB rc=$?"; tail -3 gpurun_out/r02d_nvl_n4_${MB}mb.log
  python tools/nvlink_bytes.py gpurun_out/r02d_nvl_n4_${MB}mb.csv --bucket-mb $MB --world 4 \
    > gpurun_out/r02d_nvl_n4_${MB}mb.json 2>&1; head -c 1500 gpurun_out/r02d_nvl_n4_${MB}mb.json
done
$R comm 4 0.25,1,4,16,64,256; mv gpurun_out/comm_n4.jsonl gpurun_out/r02d_comm_n4.jsonl; tail -3 gpurun_out/comm_n4.err
$R bench r02d_vgg19_b8_n4 4 --model vgg19 --batch 8 --no-cpu-baseline
$R bench r02d_vgg19_b8_n4_end 4 --model vgg19 --batch 8 --no-cpu-baseline --update-placement end
