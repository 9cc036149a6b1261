T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 python -m pytest tests/test_gpu_comm.py -q -m gpu -x 2>&1 | tail -25
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -25
b() { # name args...
  local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b36_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b36_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d.get('frac_of_compute_roofline'))"
}
b vgg_b8_deft --model vgg19 --batch 8
b vgg_b64 --model vgg19
b r101_b64 --model resnet101
b gpt2 --model gpt2
timeout 600 $T --master-port 29996 tools/trace_step.py --model vgg19 --batch 8 --scheme deft --out gpurun_out/tr36_deft > /dev/null 2>&1
