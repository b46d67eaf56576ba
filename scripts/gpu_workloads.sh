python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
for w in gemm_f32 pagerank conv kmeans; do
  st=10; [ $w = kmeans ] && st=3
  timeout -s KILL 600 python bench.py --workload $w --steps $st --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?
done
BENCH_GEMM_F32_KERNEL=gemm_tf32 timeout -s KILL 300 python bench.py --workload gemm_f32 --steps 10 --no-cpu-baseline > gpurun_out/bench_gemm_tf32.json 2>&1; echo tf32=$?
tail -n 3 gpurun_out/gpu_tests.log; for f in gpurun_out/bench_*.json; do echo $f; cut -c1-1500 $f; done; tail -n 5 gpurun_out/bench_*.err
