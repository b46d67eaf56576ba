python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nproc > gpurun_out/nproc.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout -s KILL 600 python -m pytest tests -q -m gpu --timeout 120 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout -s KILL 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/gemm_prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -n 3 gpurun_out/gpu_tests.log gpurun_out/bench.err
