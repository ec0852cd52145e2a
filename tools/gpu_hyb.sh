#!/bin/bash
# SpMV parity (all formats) + the power-law sweep (HYB spill change)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_scale.py -q -x -k "spmv or SpMV or hyb or HYB or config5 or config3" > gpurun_out/hyb_tests.log 2>&1
echo "rc=$?" >> gpurun_out/hyb_tests.log
timeout 900 python profiles/sweep_spmv.py 30 powerlaw8M,convdiff2000 > gpurun_out/hyb_sweep.json 2> gpurun_out/hyb_sweep.log
