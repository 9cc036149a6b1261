# ncu evidence, 1 GPU. Every ncu command runs only after the same command exited 0 without ncu.
set -x
timeout 600 python bench.py > gpurun_out/bench9_n1.json 2> gpurun_out/bench9_n1.err; echo bench rc=$?; cat gpurun_out/bench9_n1.json
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/ncu_launches_step.csv python tools/profile_step.py > gpurun_out/ncu_launch_run.log 2>&1
echo launches rc=$?
python tools/profile_step.py --eager > gpurun_out/prof_plain_eager.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:sgd_local -c 2 \
    -o gpurun_out/ncu_update python tools/profile_step.py --eager > gpurun_out/ncu_update_run.log 2>&1
echo update rc=$?
python tools/solver_bench.py --quick > gpurun_out/solver_quick.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:subset_sum -s 2 -c 2 \
    -o gpurun_out/ncu_dp python tools/solver_bench.py --quick > gpurun_out/ncu_dp_run.log 2>&1
echo dp rc=$?
python tools/solver_bench.py > gpurun_out/solver_full.jsonl 2> gpurun_out/solver_full.err
echo solver rc=$?
