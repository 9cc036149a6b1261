# 2 GPUs: executor parity (multi-bucket update kernel), placement comparison after steady-state warm-up
timeout 600 python -m pytest tests/test_gpu_executor.py -q 2>&1 | tail -3
for PL in end start; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --update-placement $PL > gpurun_out/b12_n1_$PL.json 2> gpurun_out/b12_n1_$PL.err; echo "n1 $PL rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/b12_n1_$PL.json').read().strip().splitlines()[-1]); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline','gpu_launches')}, d['config']['graphs_captured'], d['config']['warmup_steps_run'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958${#PL} bench.py --gpus 2 --update-placement $PL > gpurun_out/b12_n2_$PL.json 2> gpurun_out/b12_n2_$PL.err; echo "n2 $PL rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/b12_n2_$PL.json').read().strip().splitlines()[-1]); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline','gpu_launches')}, d['config']['graphs_captured'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['isolated'])"
done
