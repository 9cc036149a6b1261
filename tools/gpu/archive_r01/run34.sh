T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_comm.py tests/test_gpu_executor.py -q -m gpu -x 2>&1 | tail -3
b() { # name args...
  local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b34_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b34_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d.get('frac_of_compute_roofline'))"
}
b vgg_b8_deft --model vgg19 --batch 8
b vgg_b8_wfbp --model vgg19 --batch 8 --scheme wfbp
b vgg_b8_deft_bucket --model vgg19 --batch 8 --update-placement bucket
b vgg_b8_wfbp_bucket --model vgg19 --batch 8 --scheme wfbp --update-placement bucket
b vgg_b64 --model vgg19
b r101_b64 --model resnet101
timeout 600 python bench.py --model resnet101 > gpurun_out/b34_r101_n1.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b34_r101_n1.json').read().strip().splitlines()[-1]); print('r101 n1', d['value'], d.get('frac_of_compute_roofline'))"
timeout 600 $T --master-port 29997 tools/trace_step.py --model vgg19 --batch 8 --scheme wfbp --out gpurun_out/tr34_wfbp > /dev/null 2>&1
timeout 600 $T --master-port 29996 tools/trace_step.py --model vgg19 --batch 8 --scheme deft --out gpurun_out/tr34_deft > /dev/null 2>&1
