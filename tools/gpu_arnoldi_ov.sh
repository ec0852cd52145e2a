#!/bin/bash
# partially resident TMA Arnoldi: parity (8 M rows vs the reference fixture, fallbacks, config 2) and timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scale.py -q -x -k "arnoldi or config2" > gpurun_out/ov_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ov_tests.log
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_native_driver.py -q -x > gpurun_out/ov_solver.log 2>&1
echo "solver rc=$?" >> gpurun_out/ov_solver.log
timeout 600 python profiles/arnoldi_overflow.py 2830 > gpurun_out/ov_time_tma.log 2>&1
SPMVTUNE_MGS=stream timeout 600 python profiles/arnoldi_overflow.py 2830 > gpurun_out/ov_time_stream.log 2>&1
timeout 600 python profiles/arnoldi_overflow.py 2000 > gpurun_out/ov_time_c2.log 2>&1
