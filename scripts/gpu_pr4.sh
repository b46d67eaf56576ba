#!/bin/bash
python -c "from paper_2005_08466_b200 import build; build.build()" > /dev/null 2>&1
for cv in -1 -2; do
  echo "carveout env $cv"
  HCL_PR_CARVEOUT=$cv PR_VARIANTS="0:512:256:0,0:64:256:0,0:48:256:0,0:32:256:0,1:64:256:0,1:32:256:0" timeout 600 python scripts/prof_pagerank.py 2>&1 | tail -6
done
