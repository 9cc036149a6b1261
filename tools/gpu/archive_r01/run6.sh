set -x
timeout 300 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -5
for B in 32 64 128; do
  DEFT_COMM_BLOCKS=$B timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500+B)) tools/comm_bench.py --sizes-mb 4,64,256 > gpurun_out/comm2_b$B.jsonl 2>/dev/null; echo "blocks=$B"; cat gpurun_out/comm2_b$B.jsonl
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3_n1.json 2> gpurun_out/bench3_n1.err; echo rc=$?; tail -3 gpurun_out/bench3_n1.err; cat gpurun_out/bench3_n1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench3_n2.json 2> gpurun_out/bench3_n2.err; echo rc=$?; tail -3 gpurun_out/bench3_n2.err; cat gpurun_out/bench3_n2.json
