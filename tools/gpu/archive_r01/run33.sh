T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_executor.py -q -m gpu -x 2>&1 | tail -3
i=0
for S in deft wfbp; do
  i=$((i+1))
  timeout 900 $T --master-port 2989$i bench.py --gpus 4 --model vgg19 --batch 8 --scheme $S > gpurun_out/b33_vgg_${S}_8.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b33_vgg_${S}_8.json').read().strip().splitlines()[-1]); print('vgg n4 batch 8 $S', d['value'], d.get('frac_of_compute_roofline'))"
done
for M in vgg19 resnet101; do
  i=$((i+1))
  timeout 900 $T --master-port 2989$i bench.py --gpus 4 --model $M > gpurun_out/b33_${M}.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b33_${M}.json').read().strip().splitlines()[-1]); print('$M n4 default', d['value'], d.get('frac_of_compute_roofline'))"
done
timeout 600 python bench.py --model resnet101 > gpurun_out/b33_r101_n1.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b33_r101_n1.json').read().strip().splitlines()[-1]); print('r101 n1', d['value'], d.get('frac_of_compute_roofline'))"
timeout 600 $T --master-port 29899 tools/trace_step.py --model vgg19 --batch 8 --scheme wfbp --out gpurun_out/tr33_wfbp > /dev/null 2>&1
timeout 600 $T --master-port 29898 tools/trace_step.py --model vgg19 --batch 8 --scheme deft --out gpurun_out/tr33_deft > /dev/null 2>&1
