python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_gemm.py -q -m gpu --timeout 200 2>&1 | tail -2
timeout -s KILL 600 python scripts/diag_conv.py 2>&1 | tail -2
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.json 2>&1; cut -c1-900 gpurun_out/bench_q.json
