#!/bin/bash
# single-GPU CG with the x update moved into the p pass: CG parity (unit, native driver, BASELINE scale) and config 1/3 timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_native_driver.py -q -x > gpurun_out/cr_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/cr_tests.log
timeout 1200 python -m pytest tests/test_gpu_scale.py -q -x -k "config1_cg or config3_cg" > gpurun_out/cr_scale.log 2>&1
echo "scale rc=$?" >> gpurun_out/cr_scale.log
timeout 900 python profiles/config_details.py config1 config3 > gpurun_out/cr_details.log 2>&1
