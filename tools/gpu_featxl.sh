#!/bin/bash
# feature pass with extra-long rows on whole CTAs: parity (unit + BASELINE scale) and timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert_features.py tests/test_gpu_solver.py -q -x > gpurun_out/fx_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fx_tests.log
timeout 1200 python -m pytest tests/test_gpu_scale.py -q -x -k "features" > gpurun_out/fx_scale.log 2>&1
echo "scale rc=$?" >> gpurun_out/fx_scale.log
timeout 300 python profiles/features_time.py > gpurun_out/fx_time.log 2>&1
timeout 900 python profiles/async_ab.py > gpurun_out/fx_async_ab.log 2>&1
