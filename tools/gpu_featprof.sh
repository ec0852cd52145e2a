#!/bin/bash
# advisor kernels: feature pass and CSR->DIA conversion, full ncu captures on config 2 and a power-law matrix
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python profiles/features_time.py > gpurun_out/fp_features_time.log 2>&1
timeout 300 python profiles/convert_time.py > gpurun_out/fp_convert_time.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_features|k_csr_to_dia" -c 6 \
    -o gpurun_out/fp_full -f python profiles/advisor_kernels.py > gpurun_out/fp_full.log 2>&1
