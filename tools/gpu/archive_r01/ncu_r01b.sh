# 1 GPU: bench lines VGG-19 / GPT-2 N=1, then ncu (each ncu command preceded by the same command exiting 0)
timeout 900 python bench.py --model vgg19 --no-cpu-baseline > gpurun_out/b21_vgg19_n1.json 2>/dev/null; echo "vgg rc=$?"
timeout 900 python bench.py --model gpt2 --no-cpu-baseline > gpurun_out/b21_gpt2_n1.json 2>/dev/null; echo "gpt2 rc=$?"
python tools/profile_step.py > gpurun_out/p21_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/ncu21_launches_step.csv python tools/profile_step.py > gpurun_out/ncu21_l.log 2>&1
echo "launches rc=$?"
python tools/profile_step.py --eager > gpurun_out/p21_eager.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"gather_kernel|sgd_local" -c 4 \
    -o gpurun_out/ncu21_gather_update python tools/profile_step.py --eager > gpurun_out/ncu21_g.log 2>&1
echo "gather rc=$?"
python tools/solver_bench.py --quick > gpurun_out/p21_solver.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:deft_scheduler_kernel -c 2 \
    -o gpurun_out/ncu21_k5 python tools/solver_bench.py --quick > gpurun_out/ncu21_k5.log 2>&1
echo "k5 rc=$?"
