#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kmeans.py -q 2>&1 | tail -1
BENCH_KM_TC=1 timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('km', j['value'], j['ms_per_step'])"
BENCH_KM_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:accumulate -c 2 python bench.py --workload kmeans --steps 1 --warmup 3 2>&1 | grep -E "accumulate|gpu__time" | head -4
