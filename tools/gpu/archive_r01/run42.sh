T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b42_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b42_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['e2e']['value'], d['frac_of_compute_roofline'], d['config']['merge_counts'], d['config']['graph_choice'], d['config']['warmup_steps_run'], d['config']['graphs_captured'])"; }
b k250 --model resnet101 --comm-scale 250 --steps 15
b k1000 --model resnet101 --comm-scale 1000 --steps 15
b k500 --model resnet101 --comm-scale 500 --steps 15
b vgg --model vgg19
b gpt2 --model gpt2
