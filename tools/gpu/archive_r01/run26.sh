# in-step: TMA reduce-scatter (24 / 48 CTAs) vs LDG (128 CTAs), N=4
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for M in vgg19 resnet101; do
for CFG in "ldg 0" "tma 24" "tma 48"; do
  set -- $CFG; i=$((i+1))
  DEFT_RS_IMPL=$1 DEFT_RS_TMA_BLOCKS=$2 timeout 900 $T --master-port 2978$i bench.py --gpus 4 --model $M --steps 20 > gpurun_out/b26_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b26_$i.json').read().strip().splitlines()[-1]); print('$M $CFG', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'])"
done
done
