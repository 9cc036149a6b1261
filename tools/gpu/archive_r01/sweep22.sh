# BASELINE configs[4]: bucket-size sweep (1..256 MB) DeFT vs NCCL WFBP (DDP) at N=4, and the
# update-frequency sweep (comm times scaled so DeFT merges k = 1..4 iterations)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for MB in 1 4 16 64 256; do
  i=$((i+1))
  timeout 900 $T --master-port 2972$i bench.py --gpus 4 --bucket-mb $MB --steps 15 > gpurun_out/s22_deft_$MB.json 2>/dev/null
  timeout 900 $T --master-port 2973$i bench.py --gpus 4 --bucket-mb $MB --steps 15 --impl ddp > gpurun_out/s22_ddp_$MB.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/s22_deft_$MB.json').read().strip().splitlines()[-1]); r=json.loads(open('gpurun_out/s22_ddp_$MB.json').read().strip().splitlines()[-1])
print(json.dumps({'bucket_mb': $MB, 'deft': d['value'], 'deft_buckets': d['config']['buckets'], 'deft_frac': d['frac_of_compute_roofline'], 'ddp': r['value'], 'ratio': round(d['value']/r['value'],3)}))"
done
for CS in 100 250 500 1000; do
  i=$((i+1))
  timeout 900 $T --master-port 2972$i bench.py --gpus 4 --comm-scale $CS --steps 15 > gpurun_out/s22_k_$CS.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/s22_k_$CS.json').read().strip().splitlines()[-1])
print(json.dumps({'comm_scale': $CS, 'deft': d['value'], 'merge_counts': d['config']['merge_counts'], 'capacity_multiplier': d['config']['capacity_multiplier'], 'frac': d['frac_of_compute_roofline']}))"
done
