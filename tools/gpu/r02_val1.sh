#!/bin/bash
# Round-2 end validation on ONE GPU, most important first: pytest -m gpu, smoke,
# bench N=1, ncu --set full of sgd_local_kernel and of the loopback update /
# reduce-scatter kernels, the step's launch list, the reference arm.
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/r02v_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/r02v_smoke.log
timeout 600 python bench.py > gpurun_out/r02v_bench_n1.json 2> gpurun_out/r02v_bench_n1.err
echo "bench rc=$? $(tail -c 300 gpurun_out/r02v_bench_n1.json)"
timeout 240 python tools/profile_step.py > gpurun_out/r02v_ncu_sgd_local_plain.log 2>&1 && \
timeout 400 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:sgd_local_kernel -c 1 -o gpurun_out/r02v_ncu_sgd_local python tools/profile_step.py \
  > gpurun_out/r02v_ncu_sgd_local.log 2>&1
echo "ncu sgd_local rc=$?"
ncu -i gpurun_out/r02v_ncu_sgd_local.ncu-rep --page raw --csv > gpurun_out/r02v_ncu_sgd_local.raw.csv 2>&1
timeout 200 python tools/loopback_profile.py --mb 64 > gpurun_out/r02v_lb_plain.log 2>&1
echo "loopback plain rc=$?"
for k in update_allgather_tma reduce_scatter_tma; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/r02v_ncu_lb_$k python tools/loopback_profile.py --mb 64 > gpurun_out/r02v_ncu_lb_$k.log 2>&1
  echo "ncu loopback $k rc=$?"
  ncu -i gpurun_out/r02v_ncu_lb_$k.ncu-rep --page raw --csv > gpurun_out/r02v_ncu_lb_$k.raw.csv 2>&1
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02v_step_launches.csv python tools/profile_step.py > gpurun_out/r02v_step_ncu.log 2>&1
echo "launches rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/r02v_reference_n1.json 2> gpurun_out/r02v_reference_n1.err
echo "reference rc=$? $(tail -c 300 gpurun_out/r02v_reference_n1.json)"
