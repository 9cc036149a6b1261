# executor parity (1 and 2 GPUs), bench at N=1 and N=2, comm sweep at default CTAs
timeout 300 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench4_n1.json 2> gpurun_out/bench4_n1.err; echo rc=$?; grep -v Warning gpurun_out/bench4_n1.err | tail -3; cat gpurun_out/bench4_n1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench4_n2.json 2> gpurun_out/bench4_n2.err; echo rc=$?; tail -3 gpurun_out/bench4_n2.err; cat gpurun_out/bench4_n2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 tools/comm_bench.py > gpurun_out/comm4_n2.jsonl 2>/dev/null; cat gpurun_out/comm4_n2.jsonl
