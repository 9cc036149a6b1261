# BASELINE configs[4] re-measured with multi-bucket transfers: bucket-size sweep (1..256 MB)
# DeFT vs the wfbp schedule on the same executor vs NCCL DDP at N=4 (ResNet-101 bs64),
# and the update-frequency sweep (comm times scaled so DeFT merges k = 1..4 iterations)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
mkdir -p gpurun_out/sweep39
i=0
for MB in 1 4 16 64 256; do
  i=$((i+1))
  timeout 900 $T --master-port 2972$i bench.py --gpus 4 --bucket-mb $MB --steps 15 > gpurun_out/sweep39/deft_$MB.json 2>/dev/null
  timeout 900 $T --master-port 2973$i bench.py --gpus 4 --bucket-mb $MB --steps 15 --scheme wfbp > gpurun_out/sweep39/wfbp_$MB.json 2>/dev/null
  timeout 900 $T --master-port 2974$i bench.py --gpus 4 --bucket-mb $MB --steps 15 --impl ddp > gpurun_out/sweep39/ddp_$MB.json 2>/dev/null
  python -c "
import json
L=lambda f: json.loads(open(f).read().strip().splitlines()[-1])
d=L('gpurun_out/sweep39/deft_$MB.json'); w=L('gpurun_out/sweep39/wfbp_$MB.json'); r=L('gpurun_out/sweep39/ddp_$MB.json')
print(json.dumps({'bucket_mb': $MB, 'deft': d['value'], 'deft_buckets': d['config']['buckets'], 'deft_frac': d['frac_of_compute_roofline'], 'wfbp': w['value'], 'wfbp_frac': w['frac_of_compute_roofline'], 'ddp': r['value'], 'deft_vs_ddp': round(d['value']/r['value'],3)}))"
done
for CS in 100 250 500 1000; do
  i=$((i+1))
  timeout 900 $T --master-port 2975$i bench.py --gpus 4 --comm-scale $CS --steps 15 > gpurun_out/sweep39/k_$CS.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/sweep39/k_$CS.json').read().strip().splitlines()[-1])
print(json.dumps({'comm_scale': $CS, 'deft': d['value'], 'merge_counts': d['config']['merge_counts'], 'capacity_multiplier': d['config']['capacity_multiplier'], 'frac': d['frac_of_compute_roofline'], 'graph_choice': d['config']['graph_choice']}))"
done
