#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tc in 1 0; do
  BENCH_KM_TC=$tc timeout 900 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/km_tc$tc.json 2> gpurun_out/km_tc$tc.err; echo "tc=$tc rc=$?"
  python -c "import json; j=json.loads(open('gpurun_out/km_tc$tc.json').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline'], j.get('e2e'))"
done
tail -3 gpurun_out/km_tc1.err
