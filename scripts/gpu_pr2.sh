#!/bin/bash
# PageRank: tests + bench with/without degree-ordered relabelling
mkdir -p gpurun_out
python -c "from paper_2005_08466_b200 import build; build.build()" > gpurun_out/pr2_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pagerank.py -q -x > gpurun_out/pr2_tests.log 2>&1; echo "tests rc=$?"
for rl in 1 0; do
  for wn in 512 1024; do
    BENCH_PR_RELABEL=$rl BENCH_PR_WARP_NNZ=$wn timeout 600 python bench.py --workload pagerank --steps 20 --warmup 3 \
      > gpurun_out/pr2_bench_${rl}_${wn}.json 2> gpurun_out/pr2_bench_${rl}_${wn}.err; echo "bench rl=$rl wn=$wn rc=$?"
  done
done
tail -3 gpurun_out/pr2_tests.log
for f in gpurun_out/pr2_bench_*.json; do echo $f; python -c "
import json,sys; j=json.loads(open('$f').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline'])"; done
