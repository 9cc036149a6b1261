#!/bin/bash
# Round-2 end validation on ONE GPU: the driver's tiers (pytest -m gpu, smoke,
# bench N=1 both arms) + the ncu evidence (launch list of one step, --set full of
# sgd_local_kernel, --set full of the loopback update / reduce-scatter kernels).
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
tools/gpu/validate.sh r02v
timeout 900 python bench.py > gpurun_out/r02v_bench_n1.json 2> gpurun_out/r02v_bench_n1.err
echo "bench rc=$? $(tail -c 400 gpurun_out/r02v_bench_n1.json)"
timeout 900 python bench.py --impl reference > gpurun_out/r02v_reference_n1.json 2> gpurun_out/r02v_reference_n1.err
echo "reference rc=$? $(tail -c 300 gpurun_out/r02v_reference_n1.json)"
$R launches r02v_step
$R full r02v_ncu_sgd_local sgd_local_kernel
for k in update_allgather_tma reduce_scatter_tma; do
  timeout 300 python tools/loopback_profile.py --mb 64 > gpurun_out/r02v_lb_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/r02v_ncu_lb_$k python tools/loopback_profile.py --mb 64 > gpurun_out/r02v_ncu_lb_$k.log 2>&1
  echo "ncu loopback $k rc=$?"
  ncu -i gpurun_out/r02v_ncu_lb_$k.ncu-rep --page raw --csv > gpurun_out/r02v_ncu_lb_$k.raw.csv 2>&1
done
ncu -i gpurun_out/r02v_ncu_sgd_local.ncu-rep --page raw --csv > gpurun_out/r02v_ncu_sgd_local.raw.csv 2>&1
