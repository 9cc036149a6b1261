# in-step CTA budget of the comm kernels at N=2 (end placement)
for B in 16 32 64 128; do
DEFT_COMM_BLOCKS=$B timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+B)) bench.py --gpus 2 --steps 30 > gpurun_out/b13_n2_b$B.json 2> gpurun_out/b13_n2_b$B.err
python -c "import json,sys; d=json.loads(open('gpurun_out/b13_n2_b$B.json').read().strip().splitlines()[-1]); print($B, {k:d[k] for k in ('value','ms_per_step','compute_only_ms_per_step','frac_of_compute_roofline')}, d['config']['links'])"
done
