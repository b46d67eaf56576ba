#!/bin/bash
# PageRank N-GPU: fused exchange kernel vs NCCL allgather, same torchrun job shape (+ N=1 line)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N=${NGPU:-2}
timeout -s KILL 300 python bench.py --workload pagerank --steps 10 --warmup 3 > gpurun_out/pr_n1.json 2> gpurun_out/pr_n1.err; echo n1 rc=$?
python -c "import json; j=json.loads(open('gpurun_out/pr_n1.json').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['clocks'])"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513"
for x in 1 0; do
  BENCH_PR_EXCHANGE=$x timeout -s KILL 600 $TR bench.py --gpus $N --workload pagerank --steps 10 --warmup 3 > gpurun_out/pr_xch$x.json 2> gpurun_out/pr_xch$x.err; echo xch=$x rc=$?
  python -c "import json; j=json.loads(open('gpurun_out/pr_xch$x.json').read().strip().splitlines()[-1]); print(j['value'], j['unit'], j['ms_per_step'], j.get('e2e'), j['clocks'])" 2>&1 | tail -1
done
