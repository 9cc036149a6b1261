# N=4: start placement with small update CTA budgets (VGG-19, ResNet-101); GPT-2 graph choice
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for CFG in "vgg19 start 16" "vgg19 start 32" "vgg19 end 0" "resnet101 start 24" "resnet101 end 0"; do
  set -- $CFG; i=$((i+1))
  timeout 900 $T --master-port 2970$i bench.py --gpus 4 --model $1 --update-placement $2 --update-blocks $3 > gpurun_out/b19_$i.json 2>gpurun_out/b19_$i.err; python -c "import json; d=json.loads(open('gpurun_out/b19_$i.json').read().strip().splitlines()[-1]); print('$CFG', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'], d['config']['links'])"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --model gpt2 --no-cpu-baseline > gpurun_out/b19_gpt2.json 2>gpurun_out/b19_gpt2.err; python -c "import json; d=json.loads(open('gpurun_out/b19_gpt2.json').read().strip().splitlines()[-1]); print('gpt2 n1', d['value'], d['ms_per_step'], d['compute_only_ms_per_step'], d['frac_of_compute_roofline'], d['config']['graph_choice'])"
