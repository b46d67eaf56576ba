python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout -s KILL 600 python scripts/probe_workloads.py > gpurun_out/probe.log 2>&1; echo probe=$?
tail -n 30 gpurun_out/gpu_tests.log; cat gpurun_out/probe.log
