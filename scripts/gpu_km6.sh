#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kmeans.py -x -q 2>&1 | tail -1
for i in 1 2; do KM_N=67108864 timeout 300 python scripts/prof_kmeans_tc.py 2>&1 | tail -1; done
BENCH_KM_TC=1 timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/km_tc1.json 2>/dev/null
python -c "import json; j=json.loads(open('gpurun_out/km_tc1.json').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline']['kernel_ms'], j['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:kmeans_assign_tc -s 3 -c 1 python bench.py --workload kmeans --steps 1 --warmup 3 2>&1 | grep -E "dram__bytes|gpu__time" 
