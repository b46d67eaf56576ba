#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2005_08466_b200 import build; build.build()" > gpurun_out/pr3_build.log 2>&1
HCL_PR_NT=1024 HCL_PR_HOT=-1 timeout 600 python -m pytest tests/test_gpu_pagerank.py -q -x > gpurun_out/pr3_tests.log 2>&1; echo "tests(hot) rc=$?"
PR_VARIANTS="0:512:256:0,1:512:256:0,1:512:1024:-1,1:256:1024:-1,1:512:256:8192,1:256:256:12288,0:512:1024:-1,1:128:1024:-1" \
  timeout 900 python scripts/prof_pagerank.py > gpurun_out/pr3.log 2>&1; echo "prof rc=$?"
tail -2 gpurun_out/pr3_tests.log; cat gpurun_out/pr3.log
