#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_core.py -x -q 2>&1 | tail -2
K=gemm_f32x3 python scripts/c1_host.py; K=gemm_f32 python scripts/c1_host.py
for k in gemm_f32 gemm_f32x3; do
  BENCH_GEMM_F32_KERNEL=$k timeout 300 python bench.py --workload gemm_f32 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$k', j['value'], j['ms_per_step'], j['gpu_launches'])"
done
timeout 300 python bench.py 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bf16', j['value'], j['ms_per_step'], j['e2e']['value'])"
