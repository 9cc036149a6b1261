T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b41_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b41_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['e2e']['value'], round(d['e2e']['value']/d['value'],4), d['config']['links'])"; }
b vgg_c1 --model vgg19
b vgg_c8 --model vgg19 --h2d-chunks 8
b vgg_c32 --model vgg19 --h2d-chunks 32
b vgg_sm_c1 --model vgg19 --links sm
b r101_c1 --model resnet101
b r101_c8 --model resnet101 --h2d-chunks 8
b r101_sm_c1 --model resnet101 --links sm
for CS in 250 1000; do
  timeout 900 $T --master-port $((29800 + CS % 97)) bench.py --gpus 4 --comm-scale $CS --steps 15 > gpurun_out/b41_k_$CS.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/b41_k_$CS.json').read().strip().splitlines()[-1])
print(json.dumps({'comm_scale': $CS, 'deft': d['value'], 'e2e': d['e2e']['value'], 'merge_counts': d['config']['merge_counts'], 'frac': d['frac_of_compute_roofline'], 'graph_choice': d['config']['graph_choice']}))"
done
timeout 900 $T --master-port 29811 bench.py --gpus 4 --comm-scale 250 --steps 15 --eager > gpurun_out/b41_k_250_eager.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b41_k_250_eager.json').read().strip().splitlines()[-1]); print('k250 eager-only', d['value'], d['e2e']['value'])"
