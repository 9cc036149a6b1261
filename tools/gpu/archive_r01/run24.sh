T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_executor.py -q -k "start" 2>&1 | tail -2
i=0
for MB in 1 4 24.8; do
  i=$((i+1))
  timeout 900 $T --master-port 2975$i bench.py --gpus 4 --bucket-mb $MB --steps 15 > gpurun_out/s24_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/s24_$i.json').read().strip().splitlines()[-1]); print('$MB MB', d['value'], d['config']['buckets'], d['frac_of_compute_roofline'], d['ms_per_step'], d['compute_only_ms_per_step'])"
done
