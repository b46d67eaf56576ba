#!/usr/bin/env bash
# The round's profiling evidence on one GPU (gpurun -- bash scripts/profile_round.sh):
#  1. the ncu launch list of the default bench command (every launch's
#     gpu__time_duration; ncu's serialised cold-cache times: the kernels' share
#     of the step is the check, not the absolute);
#  2. one `ncu --set full` capture per dominant kernel at its BASELINE config.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_default.log 2>&1
echo "launch list rc=$?"
full() {  # name, kernel regex, skip, command...
  local name=$1 re=$2 skip=$3
  shift 3
  $NCU --set full --import-source on -k "regex:$re" -s "$skip" -c 1 -o "gpurun_out/$name" "$@" > "gpurun_out/$name.log" 2>&1
  echo "$name rc=$?"
}
case "${1:-all}" in
  all)
    full r02_gemm_bf16 gemm_tc 4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary
    full r02_conv_nhwc conv3x3_v3 4 python bench.py --workload conv --steps 1 --warmup 3 --no-cpu-baseline ;;
esac
full r02_pagerank_scatter pr_bin_scatter 4 python bench.py --workload pagerank --steps 1 --warmup 3 --no-cpu-baseline
full r02_pagerank_gather pr_bin_gather 4 python bench.py --workload pagerank --steps 1 --warmup 3 --no-cpu-baseline
full r02_kmeans_assign_tc_ordered assign_tc 2 python scripts/kmeans_assign_once.py 16777216 1
full r02_kmeans_accumulate_q16 accumulate32 0 python scripts/kmeans_assign_once.py 16777216 1
