# round-1 final refresh: default bench lines + baselines, current code
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
mkdir -p gpurun_out/final
one() { # name ngpu args...
  local n=$1 g=$2; shift 2
  if [ $g = 1 ]; then timeout 900 python bench.py "$@" > gpurun_out/final/$n.json 2> gpurun_out/final/$n.err
  else timeout 900 $T $g --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $g "$@" > gpurun_out/final/$n.json 2> gpurun_out/final/$n.err; fi
  python -c "import json; d=json.loads(open('gpurun_out/final/$n.json').read().strip().splitlines()[-1]); print('$n', d.get('value'), d.get('frac_of_compute_roofline'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'))"
}
one r101_n1 1 --model resnet101
one vgg19_n1 1 --model vgg19 --no-cpu-baseline
one gpt2_n1 1 --model gpt2 --no-cpu-baseline
one r101_n2 2 --model resnet101
one r101_n4 4 --model resnet101
one vgg19_n4 4 --model vgg19
one gpt2_n4 4 --model gpt2
one ddp_r101_n4 4 --model resnet101 --impl ddp
one ddp_vgg19_n4 4 --model vgg19 --impl ddp
one ddp_gpt2_n4 4 --model gpt2 --impl ddp
one wfbp_r101_n4 4 --model resnet101 --scheme wfbp
one wfbp_vgg19_n4 4 --model vgg19 --scheme wfbp
one vgg19_b8_n4 4 --model vgg19 --batch 8
one wfbp_vgg19_b8_n4 4 --model vgg19 --batch 8 --scheme wfbp
one ddp_vgg19_b8_n4 4 --model vgg19 --batch 8 --impl ddp
one reference_cpu 1 --impl reference --steps 2 --warmup 1
