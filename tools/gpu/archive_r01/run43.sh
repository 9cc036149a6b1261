T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
b() { local n=$1 g=$2; shift 2
  if [ $g = 1 ]; then timeout 900 python bench.py "$@" > gpurun_out/b43_$n.json 2>/dev/null
  else timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b43_$n.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/b43_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['e2e']['value'], d['frac_of_compute_roofline'], d['config']['graph_choice'])"; }
b gpt2_n4 4 --model gpt2
b gpt2_n1 1 --model gpt2 --no-cpu-baseline
b r101_n4 4 --model resnet101
timeout 900 $T --master-port 29861 tools/hw_experiment.py --out gpurun_out/hw43_vgg_b64 > gpurun_out/hw43_vgg_b64.log 2>&1; cat gpurun_out/hw43_vgg_b64/comparison.csv
timeout 900 $T --master-port 29862 tools/hw_experiment.py --batch 8 --out gpurun_out/hw43_vgg_b8 > gpurun_out/hw43_vgg_b8.log 2>&1; cat gpurun_out/hw43_vgg_b8/comparison.csv
