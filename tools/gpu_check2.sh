#!/bin/bash
# full GPU suite + feature timings (launch list)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/c2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/c2_tests.log
timeout 300 python profiles/features_time.py > gpurun_out/c2_features_time.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_features|k_popcount|k_bits_to|k_csr_to_dia" --csv \
    --log-file gpurun_out/c2_feat_launches.csv python profiles/features_time.py > gpurun_out/c2_feat_ncu.log 2>&1
