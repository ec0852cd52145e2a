#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert_features.py tests/test_gpu_solver.py -q -x > gpurun_out/adv_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/adv_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "features" > gpurun_out/adv_scale.log 2>&1
echo "scale rc=$?" >> gpurun_out/adv_scale.log
bash tools/gpu_featprof.sh
timeout 900 python profiles/async_ab.py > gpurun_out/adv_async_ab.log 2>&1
