#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
for cfg in "1 8 0" "0 8 0" "0 8 1" "0 4 1"; do
  set -- $cfg
  export HCL_GEMM_PERSIST=$1 HCL_GEMM_GROUP=$2 HCL_GEMM_ONE=$3
  timeout 300 python scripts/gemm_once.py > /dev/null 2>&1 || { echo "plain run failed $cfg"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 1 -c 1 --csv python scripts/gemm_once.py > gpurun_out/p_$1_$2.csv 2>&1
  python - "$1" "$2" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/p_{sys.argv[1]}_{sys.argv[2]}.csv")))
hdr = None
out = {}
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); out[d["Metric Name"]] = d["Metric Value"]
print("persist", sys.argv[1], "group", sys.argv[2], "one-acc", __import__("os").environ.get("HCL_GEMM_ONE"), out)
PY
done
unset HCL_GEMM_PERSIST HCL_GEMM_GROUP HCL_GEMM_ONE
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
timeout 600 python scripts/cmp_cublas.py
