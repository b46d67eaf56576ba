#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py -q -x 2>&1 | tail -2
for m in 0 1 0; do echo "conv epi mode $m"; HCL_CONV_EPI=$m timeout 300 python scripts/prof_conv.py; done
SWEEP_VARIANTS=8:0 SWEEP_ROUNDS=2 SWEEP_REPS=10 timeout 600 python scripts/sweep_gemm.py 2>&1 | tail -8
timeout 300 python bench.py --workload conv --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('conv bench', j['value'], j['ms_per_step'], j['roofline']['frac'], j['clocks'])"
