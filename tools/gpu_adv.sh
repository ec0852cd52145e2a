#!/bin/bash
# advisor kernels after the rewrite: parity tests, timings, full ncu captures; config-2 async/sequential
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert_features.py tests/test_gpu_solver.py tests/test_gpu_distributed.py -q -x > gpurun_out/adv_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/adv_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "features or generated or dia or DIA" > gpurun_out/adv_scale.log 2>&1
echo "scale rc=$?" >> gpurun_out/adv_scale.log
bash tools/gpu_featprof.sh
timeout 900 python profiles/config_details.py config2 config1 > gpurun_out/adv_details.log 2>&1
