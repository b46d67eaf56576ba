#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over a reduced GPU test
# subset (small shapes of every kernel family); run on the GPU box:
#   gpurun -- bash scripts/sanitize.sh
# Writes gpurun_out/sanitize_<tool>.log and a one-line verdict per tool.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SUBSET=(
  "tests/test_gpu_core.py::test_matmul_bitexact_digest[2-64]"
  "tests/test_gpu_core.py::test_vecadd_digest[4-100000]"
  "tests/test_gpu_core.py::test_knn_digest[4-200-20-8-5]"
  "tests/test_gpu_runtime.py::test_disjoint_partial_writes_keep_every_byte"
  "tests/test_gpu_runtime.py::test_trace_reduce_sum_tree"
  "tests/test_gpu_gemm.py::test_gemm_bf16_bf16out[256-256-64]"
  "tests/test_gpu_conv.py::test_conv_nhwc_equals_padded_path[2-16-16-True]"
  "tests/test_pagerank_bins.py::test_binned_step_bitexact_vs_fixed_oracle[opts1-2]"
  "tests/test_gpu_kmeans.py::test_tensor_filter_bitexact[20000-256-1]"
  "tests/test_gpu_pagerank.py::test_step_exchange_fused[2]"
)
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize_${tool}.log
  timeout 1500 compute-sanitizer --tool "$tool" --target-processes all --print-limit 20 --error-exitcode 99 \
    python -m pytest -q -x -p no:cacheprovider -m gpu "${SUBSET[@]}" > "$log" 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|passed|failed' "$log" | tail -2 | tr '\n' ' ')"
done
