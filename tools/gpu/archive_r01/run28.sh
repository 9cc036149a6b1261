timeout 900 python -m pytest tests/test_gpu_executor.py -q -k multi 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for IMPL in tma ldg; do
  i=$((i+1))
  DEFT_UPDATE_IMPL=$IMPL timeout 900 $T --master-port 2980$i bench.py --gpus 4 > gpurun_out/b28_r101_$IMPL.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b28_r101_$IMPL.json').read().strip().splitlines()[-1]); print('r101 n4 $IMPL', d['value'], d['frac_of_compute_roofline'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], json.dumps(d['roofline']['isolated']))"
  DEFT_UPDATE_IMPL=$IMPL timeout 900 $T --master-port 2981$i bench.py --gpus 4 --model vgg19 > gpurun_out/b28_vgg_$IMPL.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b28_vgg_$IMPL.json').read().strip().splitlines()[-1]); print('vgg n4 $IMPL', d['value'], d['frac_of_compute_roofline'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
done
