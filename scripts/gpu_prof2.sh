#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
export PR_VARIANTS="0:64:256:0" PR_ITERS=3
timeout 300 python scripts/prof_pagerank.py > gpurun_out/pr_plain3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pr_units -s 2 -c 1 -o gpurun_out/pr_prof3 python scripts/prof_pagerank.py > gpurun_out/pr_ncu3.log 2>&1; echo pr=$?
timeout 300 python scripts/prof_kmeans_tc.py > gpurun_out/km_plain5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans_assign_tc -s 1 -c 1 -o gpurun_out/km_tc_prof5 python scripts/prof_kmeans_tc.py > gpurun_out/km_ncu5.log 2>&1; echo km=$?
cat gpurun_out/pr_plain3.log gpurun_out/km_plain5.log
