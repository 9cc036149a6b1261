T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b53_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b53_$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$n', d['value'], d['frac_of_compute_roofline'], r['kernel'], r['achieved'], r['frac'], r['isolated']['update']['launches'])"; }
for M in resnet101 gpt2; do
  b ${M}_timed --model $M --start-grouping timed
  b ${M}_size --model $M
done
b vgg64_timed --model vgg19 --start-grouping timed
b vgg64_size --model vgg19
b vgg8_timed --model vgg19 --batch 8 --start-grouping timed
b vgg8_size --model vgg19 --batch 8
