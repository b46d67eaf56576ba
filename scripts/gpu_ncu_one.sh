#!/bin/bash
# one ncu --set full capture of a workload's dominant kernel: WL KREGEX [STEPS]
WL=$1; KR=$2; ST=${3:-2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --workload $WL --steps $ST --warmup 3 > gpurun_out/ncu_pre_$WL.json 2>/dev/null || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:$KR -s 3 -c 1 -o gpurun_out/ncu_$WL -f \
  python bench.py --workload $WL --steps $ST --warmup 3 > gpurun_out/ncu_$WL.log 2>&1; echo ncu rc=$?
