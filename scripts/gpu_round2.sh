python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 15 gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cut -c1-2500 gpurun_out/bench.json; tail -n 5 gpurun_out/bench.err
