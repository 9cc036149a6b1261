# bf16 + placement experiments, VGG-19 / GPT-2 bench lines
timeout 400 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -3
for PL in bucket end; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --update-placement $PL > gpurun_out/b8_r101_$PL.json 2> gpurun_out/b8_r101_$PL.err; echo "r101 $PL rc=$?"; cat gpurun_out/b8_r101_$PL.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline')}, d['roofline']['in_step_achieved'])"
done
for M in vgg19 gpt2; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --model $M --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/b8_$M.json 2> gpurun_out/b8_$M.err; echo "$M rc=$?"; tail -2 gpurun_out/b8_$M.err; cat gpurun_out/b8_$M.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 20 --warmup 5 --update-placement end > gpurun_out/b8_n2_end.json 2> gpurun_out/b8_n2_end.err; echo "n2 end rc=$?"; cat gpurun_out/b8_n2_end.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline')})"
