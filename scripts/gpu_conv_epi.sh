#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in 0 1 2 0; do echo "epi mode $m"; HCL_CONV_EPI=$m timeout 300 python scripts/prof_conv.py; done
