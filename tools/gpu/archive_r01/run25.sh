# TMA-staged reduce-scatter: correctness + CTA sweep vs the LDG kernel (2 and 4 GPUs run separately)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $T --master-port 29761 tools/comm_bench.py --check --sizes-mb 4,64,256 > gpurun_out/c25_ldg.jsonl 2>gpurun_out/c25_ldg.err; echo "ldg rc=$?"; cat gpurun_out/c25_ldg.jsonl | cut -c1-260
i=1
for B in 8 16 24 48; do
  i=$((i+1))
  DEFT_RS_IMPL=tma DEFT_RS_TMA_BLOCKS=$B timeout 300 $T --master-port 2976$i tools/comm_bench.py --check --sizes-mb 4,64,256 > gpurun_out/c25_tma$B.jsonl 2>gpurun_out/c25_tma$B.err; echo "tma $B rc=$?"; cat gpurun_out/c25_tma$B.jsonl | cut -c1-260; tail -3 gpurun_out/c25_tma$B.err
done
