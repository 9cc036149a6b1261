#!/bin/bash
# Round-end style validation on one GPU (run through gpurun):
#   GPU tests, smoke(), and smoke() under ncu (launch list of the hot path).
# usage: tools/gpu/validate.sh TAG [pytest -k expr]
TAG=${1:-val}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 "${KARG[@]}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"; tail -4 gpurun_out/${TAG}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_smoke.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_ncu_smoke.log 2>&1
echo "ncu smoke rc=$?"; tail -4 gpurun_out/${TAG}_ncu_smoke.log
python - "$TAG" <<'PY'
import csv, collections, sys, re
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/{tag}_launches_smoke.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
k = rows[hdr].index("Kernel Name")
c = collections.Counter(re.sub(r"[<(].*", "", r[k]) for r in rows[hdr + 1:] if len(r) > k)
mine = {n: v for n, v in c.items() if any(s in n for s in (
    "reduce_scatter", "update_allgather", "barrier_kernel", "ce_reduce", "sgd_local",
    "gather_kernel", "subset_sum", "deft_scheduler"))}
print("deft kernels under ncu:", mine)
PY
