# 4 GPUs at the current state: parity at W=4, ResNet-101 / VGG-19 / GPT-2 N=4 + DDP baselines
timeout 900 python -m pytest tests/test_gpu_executor.py -q -k multi 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for M in resnet101 vgg19 gpt2; do
  i=$((i+1))
  timeout 900 $T --master-port 2966$i bench.py --gpus 4 --model $M > gpurun_out/b16_$M.json 2> gpurun_out/b16_$M.err; echo "deft $M rc=$?"; cat gpurun_out/b16_$M.json | cut -c1-700
  timeout 900 $T --master-port 2967$i bench.py --gpus 4 --model $M --impl ddp > gpurun_out/b16_ddp_$M.json 2> gpurun_out/b16_ddp_$M.err; echo "ddp $M rc=$?"; cat gpurun_out/b16_ddp_$M.json
done
