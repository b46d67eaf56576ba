#!/bin/bash
# k-means: default build, GPU tests, bench line (tensor filter)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_core.py -x -q 2>&1 | tail -2
KM_N=67108864 timeout 300 python scripts/prof_kmeans_tc.py 2>&1 | tail -1
BENCH_KM_TC=1 timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/km_tc1.json 2> gpurun_out/km_tc1.err; echo rc=$?
python -c "import json; j=json.loads(open('gpurun_out/km_tc1.json').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline'], j['e2e'])"
