T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29861 tools/hw_experiment.py --out gpurun_out/hw_vgg_b64 > gpurun_out/hw_vgg_b64.log 2>&1; tail -3 gpurun_out/hw_vgg_b64.log; cat gpurun_out/hw_vgg_b64/comparison.csv
timeout 900 $T --master-port 29862 tools/hw_experiment.py --batch 8 --out gpurun_out/hw_vgg_b8 > gpurun_out/hw_vgg_b8.log 2>&1; tail -3 gpurun_out/hw_vgg_b8.log; cat gpurun_out/hw_vgg_b8/comparison.csv
i=0
for S in deft wfbp ddp; do for Bt in 8 16; do
  i=$((i+1))
  if [ $S = ddp ]; then A="--impl ddp"; else A="--scheme $S"; fi
  timeout 900 $T --master-port 2987$i bench.py --gpus 4 --model vgg19 --batch $Bt $A > gpurun_out/b31_vgg_${S}_$Bt.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b31_vgg_${S}_$Bt.json').read().strip().splitlines()[-1]); print('vgg n4 batch $Bt $S', d['value'], d.get('frac_of_compute_roofline'), d['config'].get('merge_counts'))"
done; done
