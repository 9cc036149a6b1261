#!/bin/bash
# one GPU: the profiler partition test, three times
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 200 python -m pytest tests/test_gpu_loopback.py -q -m gpu -k measure_profile > gpurun_out/r02n_$i.log 2>&1
  echo "run $i rc=$? $(tail -1 gpurun_out/r02n_$i.log)"
done
