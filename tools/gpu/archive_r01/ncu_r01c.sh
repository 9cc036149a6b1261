# end-of-round ncu refresh, 1 GPU; every ncu command only after the same command exited 0
python tools/nvls_probe.py 2>&1 | tail -8
python tools/profile_step.py > gpurun_out/prof_plain_c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/ncu_launches_step_c.csv python tools/profile_step.py > gpurun_out/ncu_launch_run_c.log 2>&1
echo launches rc=$?
python tools/profile_step.py --eager > gpurun_out/prof_plain_eager_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:sgd_local -c 1 \
    -o gpurun_out/ncu_update_c python tools/profile_step.py --eager > gpurun_out/ncu_update_run_c.log 2>&1
echo update rc=$?
ncu -i gpurun_out/ncu_update_c.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/ncu_update_c_raw.csv 2>&1
echo raw rc=$?
