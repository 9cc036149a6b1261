timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/b23_n1.json 2>gpurun_out/b23_n1.err; echo "n1 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/b23_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'], d['gpu_launches'], d['roofline']['traffic'], d['solver'])"
for CS in 1000; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 2 --comm-scale $CS --steps 15 > gpurun_out/b23_k$CS.json 2>gpurun_out/b23_k$CS.err; python -c "import json; d=json.loads(open('gpurun_out/b23_k$CS.json').read().strip().splitlines()[-1]); print('cs $CS', d['value'], d['frac_of_compute_roofline'], d['config']['merge_counts'], d['config']['graph_choice'])"
done
