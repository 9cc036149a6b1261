# 4 GPUs, defaults: whole GPU suite, smoke, scaling lines
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/b20_r101_n1.json 2> gpurun_out/b20_r101_n1.err; echo "n1 rc=$?"
i=0
for N in 2 4; do
  i=$((i+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$i bench.py --gpus $N > gpurun_out/b20_r101_n$N.json 2> gpurun_out/b20_r101_n$N.err; echo "n$N rc=$?"
done
for M in vgg19 gpt2; do
  i=$((i+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$i bench.py --gpus 4 --model $M > gpurun_out/b20_${M}_n4.json 2> gpurun_out/b20_${M}_n4.err; echo "$M n4 rc=$?"
done
for f in gpurun_out/b20_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'], d['e2e']['value'], d['config']['update_placement'], d['config']['graph_choice'])"; done
