#!/bin/bash
# reusable advisor threads: solver tests, config-4 suite (B200 models), config-2 async A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_convert_features.py tests/test_gpu_native_driver.py -q -x > gpurun_out/at_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/at_tests.log
timeout 900 python profiles/async_ab.py > gpurun_out/at_async_ab.log 2>&1
timeout 1500 python -m paper_2411_10143_b200 suite --models paper_2411_10143_b200/models/b200 --out gpurun_out/suite_at > gpurun_out/suite_at.log 2>&1
python -m paper_2411_10143_b200 report gpurun_out/suite_at --out gpurun_out/suite_at.csv > gpurun_out/suite_at.txt 2>&1
