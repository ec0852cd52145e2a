#!/bin/bash
# ELL/LibC compile-time strides + vectorised fp32 DIA: SpMV parity, fp32/fp64 sweeps
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_native_driver.py -q -x > gpurun_out/sp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sp_tests.log
SWEEP_DTYPE=f32 timeout 900 python profiles/sweep_spmv.py 30 poisson1024,convdiff2000 > gpurun_out/sw_f32c.json 2> gpurun_out/sw_f32c.log
timeout 900 python profiles/sweep_spmv.py 30 poisson1024,convdiff2000 > gpurun_out/sw_f64c.json 2> gpurun_out/sw_f64c.log
