# VGG-19 N=4: link choice; GPT-2 N=1 with automatic graph choice
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for L in both ce sm; do
  i=$((i+1))
  timeout 900 $T --master-port 2969$i bench.py --gpus 4 --model vgg19 --links $L > gpurun_out/b18_vgg_$L.json 2>gpurun_out/b18_vgg_$L.err; python -c "import json; d=json.loads(open('gpurun_out/b18_vgg_$L.json').read().strip().splitlines()[-1]); print('vgg n4 $L', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'], d['config']['links'], d['config']['graph_choice'])"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --model gpt2 --no-cpu-baseline > gpurun_out/b18_gpt2.json 2>gpurun_out/b18_gpt2.err; python -c "import json; d=json.loads(open('gpurun_out/b18_gpt2.json').read().strip().splitlines()[-1]); print('gpt2 n1', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['compute_only_modes'], d['frac_of_compute_roofline'], d['config']['graph_choice'])"
