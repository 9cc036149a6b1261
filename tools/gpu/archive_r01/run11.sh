# full GPU suite (2 GPUs), smoke, placement comparison at N=1 and N=2
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -12
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for PL in end start; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --update-placement $PL > gpurun_out/b11_n1_$PL.json 2> gpurun_out/b11_n1_$PL.err; echo "n1 $PL rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/b11_n1_$PL.json').read().strip().splitlines()[-1]); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline','gpu_launches')}, d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957${#PL} bench.py --gpus 2 --update-placement $PL > gpurun_out/b11_n2_$PL.json 2> gpurun_out/b11_n2_$PL.err; echo "n2 $PL rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/b11_n2_$PL.json').read().strip().splitlines()[-1]); print({k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline','gpu_launches')}, d['e2e']['value'])"
done
