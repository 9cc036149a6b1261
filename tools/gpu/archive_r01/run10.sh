# 4 GPUs: parity at W=4, bench N=4 (+ measured profile), DDP baseline, comm sweep
nvidia-smi topo -m | head -6
timeout 400 python -m pytest tests/test_gpu_executor.py -x -q -k multi 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $T --master-port 29561 bench.py --gpus 4 --dump-profile gpurun_out/profile_resnet101_w4.json > gpurun_out/b10_n4.json 2> gpurun_out/b10_n4.err; echo "deft n4 rc=$?"; cat gpurun_out/b10_n4.json
timeout 600 $T --master-port 29562 bench.py --gpus 4 --impl ddp > gpurun_out/b10_ddp_n4.json 2> gpurun_out/b10_ddp_n4.err; echo "ddp n4 rc=$?"; cat gpurun_out/b10_ddp_n4.json
timeout 300 $T --master-port 29563 tools/comm_bench.py > gpurun_out/comm10_n4.jsonl 2>/dev/null; cat gpurun_out/comm10_n4.jsonl
timeout 600 $T --master-port 29564 bench.py --gpus 4 --model vgg19 --dump-profile gpurun_out/profile_vgg19_w4.json > gpurun_out/b10_vgg_n4.json 2> gpurun_out/b10_vgg_n4.err; echo "vgg n4 rc=$?"; cat gpurun_out/b10_vgg_n4.json
