#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert_features.py -q -x > gpurun_out/f3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/f3_tests.log
timeout 300 python profiles/features_time.py > gpurun_out/f3_features_time.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_features|k_csr_to_dia" --csv \
    --log-file gpurun_out/f3_feat_launches.csv python profiles/features_time.py > gpurun_out/f3_feat_ncu.log 2>&1
