T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
DEFT_UPDATE_TMA_STAGES=6 timeout 900 python -m pytest tests/test_gpu_executor.py -q -m gpu -x -k multi 2>&1 | tail -1
i=0
for S in 3 6; do
  i=$((i+1))
  DEFT_UPDATE_TMA_STAGES=$S timeout 300 $T --master-port 2951$i tools/comm_bench.py --sizes-mb 16,64,256 --update-blocks 32 > gpurun_out/c51_$S.jsonl 2>/dev/null
  grep "^{" gpurun_out/c51_$S.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('upd stages $S', d['bucket_mb'], 'upd_ag busbw', d['upd_ag_busbw_gbs'])"
done
b() { local n=$1; shift
  timeout 900 $T --master-port $((29900 + RANDOM % 90)) bench.py --gpus 4 "$@" > gpurun_out/b51_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b51_$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$n', d['value'], d['frac_of_compute_roofline'], r['kernel'], r['achieved'], r['frac'])"; }
DEFT_UPDATE_TMA_STAGES=6 b r101_s6 --model resnet101
b r101_s3 --model resnet101
DEFT_UPDATE_TMA_STAGES=6 b gpt2_s6 --model gpt2
