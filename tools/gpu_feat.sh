#!/bin/bash
# feature pass (ring + device cancel word), DIA conversion from cached offsets, TMA Arnoldi gate
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert_features.py tests/test_gpu_solver.py -q -x > gpurun_out/ft_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ft_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "tma_arnoldi or features" > gpurun_out/ft_scale.log 2>&1
echo "scale rc=$?" >> gpurun_out/ft_scale.log
timeout 300 python profiles/features_time.py > gpurun_out/ft_features_time.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_features|k_popcount|k_bits_to|k_csr_to_dia|k_diag_bits" --csv \
    --log-file gpurun_out/ft_feat_launches.csv python profiles/features_time.py > gpurun_out/ft_feat_ncu.log 2>&1
