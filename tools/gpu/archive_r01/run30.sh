T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 300 $T --master-port 29831 tools/comm_bench.py --sizes-mb 1,16,64 --check > gpurun_out/c30.jsonl 2>/dev/null; grep -c check_err gpurun_out/c30.jsonl
i=0
for M in resnet101 gpt2; do for B in 16 32; do
  i=$((i+1))
  timeout 900 $T --master-port 2984$i bench.py --gpus 4 --model $M --update-blocks $B > gpurun_out/b30_${M}_$B.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b30_${M}_$B.json').read().strip().splitlines()[-1]); print('$M n4 blocks $B', d['value'], d['frac_of_compute_roofline'], d['roofline']['achieved'], d['roofline']['frac'])"
done; done
for S in wfbp priority; do for M in resnet101 vgg19; do
  i=$((i+1))
  timeout 900 $T --master-port 2985$i bench.py --gpus 4 --model $M --scheme $S > gpurun_out/b30_${M}_$S.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b30_${M}_$S.json').read().strip().splitlines()[-1]); print('$M n4 $S', d['value'], d['frac_of_compute_roofline'], d['config']['buckets'])"
done; done
