T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_executor.py -q -m gpu -x 2>&1 | tail -3
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b45_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b45_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['e2e']['value'], d['frac_of_compute_roofline'])"; }
b vgg8_start --model vgg19 --batch 8
b vgg8_bucket --model vgg19 --batch 8 --update-placement bucket
b vgg64_start --model vgg19
b vgg64_bucket --model vgg19 --update-placement bucket
b r101_start --model resnet101
b r101_bucket --model resnet101 --update-placement bucket
b gpt2_bucket --model gpt2 --update-placement bucket
