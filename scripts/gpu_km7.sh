#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kmeans.py -x -q 2>&1 | tail -2
for d in 0 16 4 2; do HCL_KM_DBG=$d KM_N=67108864 timeout 300 python scripts/prof_kmeans_tc.py 2>&1 | tail -2 | sed "s/^/dbg=$d /"; done
