T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_executor.py -q -m gpu -x 2>&1 | tail -1
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b54_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b54_$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$n', d['value'], d['frac_of_compute_roofline'], d['e2e']['value'], r['kernel'], r['achieved'], r['frac'], r['isolated']['update']['launches'])"; }
b r101 --model resnet101
b vgg64 --model vgg19
b vgg8 --model vgg19 --batch 8
b gpt2 --model gpt2
