#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv.py -q > /tmp/t.log 2>&1; tail -1 /tmp/t.log
for m in 0 4 0 4; do echo "epi $m"; HCL_CONV_EPI=$m timeout 300 python scripts/prof_conv.py; done
for m in 0 4; do
  HCL_CONV_EPI=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:conv3x3_v2 -s 1 -c 1 --csv python scripts/prof_conv.py 2>/dev/null | grep -E "dram|gpu__time|cycles_elapsed" | cut -d, -f13,15
done
