# end-of-round validation of the committed tree
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('build+smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/b47_n1.json 2> gpurun_out/b47_n1.err; echo n1 rc=$?; tail -1 gpurun_out/b47_n1.json | cut -c1-300
timeout 900 $T 2 --master-addr 127.0.0.1 --master-port 29471 bench.py --gpus 2 > gpurun_out/b47_n2.json 2> gpurun_out/b47_n2.err; echo n2 rc=$?; tail -1 gpurun_out/b47_n2.json | cut -c1-200
timeout 900 $T 4 --master-addr 127.0.0.1 --master-port 29472 bench.py --gpus 4 > gpurun_out/b47_n4.json 2> gpurun_out/b47_n4.err; echo n4 rc=$?; tail -1 gpurun_out/b47_n4.json | cut -c1-200
timeout 900 $T 4 --master-addr 127.0.0.1 --master-port 29473 bench.py --gpus 4 --impl reference > gpurun_out/b47_ref_n4.json 2> gpurun_out/b47_ref_n4.err; echo ref4 rc=$?; cat gpurun_out/b47_ref_n4.json | cut -c1-200
