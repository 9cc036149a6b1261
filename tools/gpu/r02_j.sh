#!/bin/bash
# 2-GPU box, final check of the last changes: W-dependent update chunk (loopback
# parity W = 2/4/8 + the experiment test), smoke, bench N=1 and N=2 (clock load
# padding with collectives), graphed DDP N=2 (exit path).
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_experiment.py -q -m gpu -x \
  > gpurun_out/r02j_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02j_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/r02j_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/r02j_r101_n1.json 2> gpurun_out/r02j_r101_n1.err
echo "bench n1 rc=$? $(tail -c 200 gpurun_out/r02j_r101_n1.json)"
timeout 400 $T --master-port 29871 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r02j_r101_n2.json 2> gpurun_out/r02j_r101_n2.err
echo "bench n2 rc=$? $(tail -c 200 gpurun_out/r02j_r101_n2.json)"
timeout 300 $T --master-port 29872 bench.py --gpus 2 --impl ddp --ddp-graphs > gpurun_out/r02j_ddpgraph_r101_n2.json 2> gpurun_out/r02j_ddpgraph_r101_n2.err
echo "ddp graph n2 rc=$? $(tail -c 200 gpurun_out/r02j_ddpgraph_r101_n2.json)"
