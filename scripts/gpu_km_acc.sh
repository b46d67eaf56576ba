#!/bin/bash
# k-means accumulate: TMA-streamed kernel vs the register-pipelined one
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kmeans.py -x -q 2>&1 | tail -3
for b in 1; do
  HCL_KM_ACC_BULK=$b BENCH_KM_TC=1 timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/km_acc$b.json 2>/dev/null
  python -c "import json; j=json.loads(open('gpurun_out/km_acc$b.json').read().strip().splitlines()[-1]); print('bulk=$b', j['value'], j['ms_per_step'], j['roofline']['kernel_ms'])"
done
HCL_KM_ACC_BULK=1 BENCH_KM_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:accumulate -c 4 --csv --log-file gpurun_out/km_acc_launches.csv python bench.py --workload kmeans --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu rc=$?
