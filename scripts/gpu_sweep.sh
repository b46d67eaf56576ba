#!/bin/bash
# GEMM raster-group / L2-promotion sweep + fp32 kernels, then DRAM bytes per launch under ncu.
set -x
mkdir -p gpurun_out
python -c "from paper_2005_08466_b200 import build; build.build()" > gpurun_out/sweep_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/sweep_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python scripts/sweep_gemm.py > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
export SWEEP_REPS=1 SWEEP_ROUNDS=1 SWEEP_F32_BIG=0
if timeout 600 python scripts/sweep_gemm.py > gpurun_out/sweep1.log 2>&1; then
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:gemm_tc --clock-control none --csv --log-file gpurun_out/sweep_dram.csv \
    python scripts/sweep_gemm.py > gpurun_out/sweep_ncu.log 2>&1; echo "ncu rc=$?"
fi
tail -5 gpurun_out/sweep_tests.log; cat gpurun_out/sweep.log
