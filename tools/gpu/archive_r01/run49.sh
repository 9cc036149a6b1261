T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
DEFT_RS_TMA_STAGES=6 timeout 400 python -m pytest tests/test_gpu_comm.py -q -m gpu 2>&1 | tail -1
i=0
for S in 4 6; do for B in 24 32; do
  i=$((i+1))
  DEFT_RS_TMA_STAGES=$S DEFT_RS_TMA_BLOCKS=$B timeout 300 $T --master-port 2949$i tools/comm_bench.py --sizes-mb 16,64,256 > gpurun_out/c49_${S}_$B.jsonl 2>/dev/null
  grep "^{" gpurun_out/c49_${S}_$B.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('stages $S blocks $B', d['bucket_mb'], 'rs_sm busbw', d['rs_sm_busbw_gbs'])"
done; done
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b49_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b49_$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$n', d['value'], d['frac_of_compute_roofline'], r['kernel'], r['achieved'], r['frac'])"; }
DEFT_RS_TMA_STAGES=6 b vgg64_s6 --model vgg19
DEFT_RS_TMA_STAGES=6 b vgg8_s6 --model vgg19 --batch 8
b vgg64_s4 --model vgg19
