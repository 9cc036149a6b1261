T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_executor.py -q -m gpu -x 2>&1 | tail -2
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b46_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b46_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['e2e']['value'], d['frac_of_compute_roofline'])"; }
b vgg8 --model vgg19 --batch 8
b vgg64 --model vgg19
b r101 --model resnet101
b gpt2 --model gpt2
b vgg8_wfbp --model vgg19 --batch 8 --scheme wfbp
