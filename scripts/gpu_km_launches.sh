#!/bin/bash
# k-means iteration: per-kernel launch list (ncu, durations only) after a clean run
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
BENCH_KM_TC=1 timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/km_tc1.json 2> gpurun_out/km_tc1.err || exit 1
tail -c 400 gpurun_out/km_tc1.json
BENCH_KM_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/km_launches.csv python bench.py --workload kmeans --steps 1 --warmup 3 > gpurun_out/km_ncu.log 2>&1; echo ncu rc=$?
