T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for B in 16 32 64 128; do
  i=$((i+1))
  timeout 300 $T --master-port 2982$i tools/comm_bench.py --sizes-mb 16,64,256 --update-blocks $B > gpurun_out/c29_$B.jsonl 2>/dev/null
  grep "^{" gpurun_out/c29_$B.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('blocks $B', d['bucket_mb'], 'upd_ag', d['upd_ag_ms'], d['upd_ag_busbw_gbs'], 'deft vs nccl+sgd', d['deft_vs_nccl_ar_sgd'])"
done
for B in 32 64; do
  i=$((i+1))
  timeout 900 $T --master-port 2982$i bench.py --gpus 4 --model vgg19 --update-blocks $B > gpurun_out/b29_vgg_$B.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b29_vgg_$B.json').read().strip().splitlines()[-1]); print('vgg n4 blocks $B', d['value'], d['frac_of_compute_roofline'], d['roofline']['achieved'], d['roofline']['frac'])"
done
