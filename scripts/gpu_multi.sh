#!/bin/bash
# N-GPU check: all GPU tests (incl. tests/test_gpu_multi.py over distinct GPUs) + torchrun benches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N=${NGPU:-2}
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x > gpurun_out/multi_tests.log 2>&1; echo tests=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout -s KILL 600 $TR bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/multi_gemm.json 2> gpurun_out/multi_gemm.err; echo gemm=$?
timeout -s KILL 600 $TR bench.py --gpus $N --workload pagerank --steps 10 --warmup 3 > gpurun_out/multi_pr.json 2> gpurun_out/multi_pr.err; echo pr=$?
timeout -s KILL 600 $TR bench.py --gpus $N --workload conv --steps 10 --warmup 3 > gpurun_out/multi_conv.json 2> gpurun_out/multi_conv.err; echo conv=$?
timeout -s KILL 900 $TR bench.py --gpus $N --workload kmeans --steps 3 --warmup 3 > gpurun_out/multi_km.json 2> gpurun_out/multi_km.err; echo km=$?
timeout -s KILL 300 $TR bench.py --gpus $N --impl reference --steps 3 --warmup 1 > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err; echo ref=$?
tail -n 3 gpurun_out/multi_tests.log
for f in gpurun_out/multi_*.json; do echo $f; cut -c1-900 $f; done; tail -n 4 gpurun_out/multi_*.err
