T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $T --master-port 29881 tools/trace_step.py --model vgg19 --batch 8 --scheme deft --out gpurun_out/tr_deft > gpurun_out/tr_deft.log 2>&1; echo deft $?
timeout 600 $T --master-port 29882 tools/trace_step.py --model vgg19 --batch 8 --scheme wfbp --out gpurun_out/tr_wfbp > gpurun_out/tr_wfbp.log 2>&1; echo wfbp $?
ls -la gpurun_out/tr_deft gpurun_out/tr_wfbp
