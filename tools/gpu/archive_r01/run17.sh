# GPT-2 graph vs eager vs DDP(N=1); VGG-19 start vs end at N=4
export CUDA_VISIBLE_DEVICES=0
for A in "" "--eager"; do
timeout 900 python bench.py --model gpt2 --no-cpu-baseline $A > gpurun_out/b17_gpt2$A.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b17_gpt2$A.json').read().strip().splitlines()[-1]); print('gpt2 $A', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'])"
done
timeout 900 python bench.py --model gpt2 --impl ddp > gpurun_out/b17_gpt2_ddp.json 2>/dev/null; cat gpurun_out/b17_gpt2_ddp.json | cut -c1-300
python - <<'PY'
import torch, time, sys
sys.path.insert(0, '.')
import bench
m = bench.build_model('gpt2', torch.device('cuda'))
b = bench.make_batch('gpt2', 16, 'cuda')
lf = bench.loss_fn_for('gpt2')
from torch.nn.attention import sdpa_kernel, SDPBackend
print('attn impl', m.config._attn_implementation)
def step():
    l = lf(m, b); l.backward()
for _ in range(3): step()
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): step()
torch.cuda.synchronize(); print('eager fwd+bwd ms', (time.perf_counter()-t)/5*1e3)
PY
unset CUDA_VISIBLE_DEVICES
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29681 bench.py --gpus 4 --model vgg19 --update-placement start > gpurun_out/b17_vgg_start.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b17_vgg_start.json').read().strip().splitlines()[-1]); print('vgg n4 start', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'])"
timeout 900 $T --master-port 29682 bench.py --gpus 4 --update-placement start > gpurun_out/b17_r101_start.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b17_r101_start.json').read().strip().splitlines()[-1]); print('r101 n4 start', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'])"
