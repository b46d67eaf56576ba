#!/bin/bash
# all GPU tests + fp32 GEMM timings after the tile-shape change
mkdir -p gpurun_out
python -c "from paper_2005_08466_b200 import build; build.build()" > gpurun_out/q2_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/q2_tests.log 2>&1; echo "tests rc=$?"
SWEEP_VARIANTS=8:0 SWEEP_ROUNDS=1 SWEEP_REPS=5 timeout 900 python scripts/sweep_gemm.py > gpurun_out/q2_sweep.log 2>&1; echo "sweep rc=$?"
tail -3 gpurun_out/q2_tests.log; cat gpurun_out/q2_sweep.log
