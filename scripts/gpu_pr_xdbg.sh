#!/bin/bash
# where the N-GPU PageRank step time goes: exchange diagnostics (wrong ranks for 1/2)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
N=${NGPU:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515"
for x in 0 1 2; do
  BENCH_PR_XCH_DBG=$x timeout -s KILL 600 $TR bench.py --gpus $N --workload pagerank --steps 20 --warmup 3 > gpurun_out/pr_xdbg$x.json 2>/dev/null
  python -c "import json; j=json.loads(open('gpurun_out/pr_xdbg$x.json').read().strip().splitlines()[-1]); print('dbg=$x', j['value'], j['ms_per_step'], j['roofline']['kernel_ms'])"
done
