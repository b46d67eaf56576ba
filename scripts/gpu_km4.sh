#!/bin/bash
# k-means tensor-filter variants: scan groups / list slots / chunk width (HCL_KT_GROUPS / HCL_KT_LIST / HCL_KT_CW)
for v in "4 4 128" "4 4 256" "2 8 128"; do
  set -- $v
  touch paper_2005_08466_b200/csrc/k_kmeans_tc.cu
  HCL_NVCC_EXTRA="-DHCL_KT_GROUPS=$1 -DHCL_KT_LIST=$2 -DHCL_KT_CW=$3" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "== $v"; timeout 600 python -m pytest tests/test_gpu_kmeans.py -x -q 2>&1 | tail -1
  for d in 0 16 4 2; do
    echo "== $v dbg=$d"; HCL_KM_DBG=$d KM_N=67108864 timeout 300 python scripts/prof_kmeans_tc.py 2>&1 | tail -2
  done
done
