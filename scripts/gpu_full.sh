#!/bin/bash
# Round check: all GPU tests + smoke, default bench + reference arm, every workload, ncu launch list
# of the default bench and one full capture of the GEMM launch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout -s KILL 1500 python -m pytest tests -q -m gpu --timeout 300 --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for w in gemm_f32 pagerank conv kmeans; do
  st=10; [ $w = kmeans ] && st=3
  timeout -s KILL 600 python bench.py --workload $w --steps $st --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?
done
BENCH_GEMM_F32_KERNEL=gemm_f32x3 timeout -s KILL 300 python bench.py --workload gemm_f32 --steps 10 --warmup 3 > gpurun_out/bench_gemm_f32x3.json 2> gpurun_out/bench_gemm_f32x3.err; echo f32x3=$?
BENCH_GEMM_F32_KERNEL=gemm_f32x3 BENCH_GEMM_F32_S=16384 timeout -s KILL 600 python bench.py --workload gemm_f32 --steps 5 --warmup 3 > gpurun_out/bench_gemm_f32x3_16k.json 2> gpurun_out/bench_gemm_f32x3_16k.err; echo f32x3_16k=$?
if [ -s gpurun_out/bench.json ]; then
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo ncu_launches=$?
fi
tail -n 3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log | tail -2
for f in gpurun_out/bench*.json; do echo $f; cut -c1-2500 $f; done
