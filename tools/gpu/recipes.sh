#!/bin/bash
# Parameterized gpurun recipes behind profiles/ (run from the repo root on the
# GPU box, e.g.  gpurun --gpus 4 -- tools/gpu/recipes.sh bench r101_n4 4 --model resnet101).
# Outputs under gpurun_out/.  Every ncu recipe runs the same command without ncu
# first and only profiles it if that exited 0.
#
#   bench TAG N [bench.py args]        one bench line (torchrun for N > 1) -> TAG.json
#   comm N [SIZES_MB]                  tools/comm_bench.py --check -> comm_nN.jsonl
#   update_w1                          tools/update_bench.py (sgd_local variants, GPU 0)
#   launches TAG [profile_step args]   ncu launch list of one step (1 GPU) -> TAG_launches.csv
#   full TAG KERNEL_REGEX [args]       ncu --set full of one launch of KERNEL -> TAG.ncu-rep + raw csv
#   trace TAG N [trace_step args]      torch.profiler timeline of steady-state steps
#   validate TAG                       tools/gpu/validate.sh (GPU tests, smoke, smoke under ncu)
#   sass                               tools/sass_summary.py (no GPU needed)
set -u
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port() { echo $((29500 + RANDOM % 400)); }
cmd=${1:-}; shift || true
case "$cmd" in
  bench)
    tag=$1 n=$2; shift 2
    if [ "$n" = 1 ]; then timeout 900 python bench.py "$@" > gpurun_out/$tag.json 2> gpurun_out/$tag.err
    else timeout 900 $T --nproc-per-node $n --master-port $(port) bench.py --gpus $n "$@" \
           > gpurun_out/$tag.json 2> gpurun_out/$tag.err; fi
    echo "$tag rc=$? $(tail -c 300 gpurun_out/$tag.json)";;
  comm)
    n=$1 sizes=${2:-0.25,1,4,16,64,256}
    timeout 900 $T --nproc-per-node $n --master-port $(port) tools/comm_bench.py --sizes-mb $sizes \
      --check > gpurun_out/comm_n$n.jsonl 2> gpurun_out/comm_n$n.err
    echo "comm n=$n rc=$?";;
  update_w1)
    CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/update_bench.py "$@" > gpurun_out/update_w1.jsonl 2>&1
    echo "update_w1 rc=$?";;
  launches)
    tag=$1; shift
    python tools/profile_step.py "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
    echo "launches $tag rc=$?";;
  full)
    tag=$1 k=$2; shift 2
    python tools/profile_step.py "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -c 1 \
      -o gpurun_out/$tag python tools/profile_step.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
    echo "full $tag rc=$?"
    ncu -i gpurun_out/$tag.ncu-rep --page raw --csv --metrics \
      gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/${tag}_raw.csv 2>&1;;
  trace)
    tag=$1 n=$2; shift 2
    timeout 900 $T --nproc-per-node $n --master-port $(port) tools/trace_step.py --out gpurun_out/$tag "$@" \
      > gpurun_out/$tag.log 2>&1
    echo "trace $tag rc=$?";;
  validate) tools/gpu/validate.sh "$@";;
  sass) python tools/sass_summary.py;;
  *) sed -n 2,20p "$0"; exit 2;;
esac
