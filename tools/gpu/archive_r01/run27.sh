timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $T --master-port 29791 tools/comm_bench.py --check > gpurun_out/c27.jsonl 2>/dev/null; grep "^{" gpurun_out/c27.jsonl | cut -c1-200
timeout 900 $T --master-port 29792 bench.py --gpus 4 > gpurun_out/b27_n4.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b27_n4.json').read().strip().splitlines()[-1]); print('r101 n4', d['value'], d['frac_of_compute_roofline'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
