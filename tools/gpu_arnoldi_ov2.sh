#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scale.py -q -x -k "arnoldi" > gpurun_out/ov2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ov2_tests.log
timeout 600 python profiles/arnoldi_overflow.py 2830 > gpurun_out/ov2_time_tma.log 2>&1
timeout 600 python profiles/arnoldi_overflow.py 3500 > gpurun_out/ov2_time_12M.log 2>&1
SPMVTUNE_MGS=stream timeout 600 python profiles/arnoldi_overflow.py 3500 > gpurun_out/ov2_time_12M_stream.log 2>&1
