#!/bin/bash
# Final state, one GPU: the driver's GPU tiers (pytest -m gpu, smoke, bench N=1).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/r02zzz_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02zzz_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zzz_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/r02zzz_smoke.log
timeout 400 python bench.py > gpurun_out/r02zzz_bench_n1.json 2> gpurun_out/r02zzz_bench_n1.err
echo "bench rc=$? $(tail -c 120 gpurun_out/r02zzz_bench_n1.json)"
