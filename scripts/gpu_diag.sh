python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 300 python scripts/diag_gemm.py > gpurun_out/diag.log 2>&1; echo diag=$?
timeout -s KILL 300 python -m pytest tests/test_gpu_core.py -q -m gpu --timeout 120 -k migration > gpurun_out/core.log 2>&1; echo core=$?
cat gpurun_out/diag.log; tail -n 3 gpurun_out/core.log
