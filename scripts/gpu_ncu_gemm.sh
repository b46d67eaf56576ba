#!/bin/bash
# final ncu --set full capture of the headline GEMM launch (after the plain bench exited 0)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_pre_gemm.json 2>/dev/null || exit 1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 6 -c 1 -o gpurun_out/ncu_gemm -f \
  python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_gemm.log 2>&1; echo ncu rc=$?
