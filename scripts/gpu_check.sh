set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout -s KILL 400 python -m pytest tests/test_gpu_core.py -q -m gpu --timeout 120 > gpurun_out/core.log 2>&1; echo core=$?
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -m gpu --timeout 120 > gpurun_out/gemm.log 2>&1; echo gemm=$?
tail -3 gpurun_out/core.log gpurun_out/gemm.log gpurun_out/smoke.log
