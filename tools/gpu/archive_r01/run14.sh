true
python tools/solver_bench.py > gpurun_out/solver14.jsonl 2> gpurun_out/solver14.err; echo solver rc=$?; cat gpurun_out/solver14.jsonl; tail -3 gpurun_out/solver14.err
