timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/b15_n1.json 2> gpurun_out/b15_n1.err; echo "n1 rc=$?"; cat gpurun_out/b15_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 2 > gpurun_out/b15_n2.json 2> gpurun_out/b15_n2.err; echo "n2 rc=$?"; cat gpurun_out/b15_n2.json
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > gpurun_out/b15_ref.json 2> gpurun_out/b15_ref.err; echo "ref rc=$?"; cat gpurun_out/b15_ref.json
