#!/bin/bash
# full ncu captures of the config-3 row kernels after dynamic tile claims (HYB spill, CSR/LibB)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows_pipe -s 1 -c 1 -o gpurun_out/pl_after_hyb -f python profiles/run_spmv.py powerlaw8M HYB/LibA 3 > gpurun_out/pl_after_hyb.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows_pipe -s 1 -c 1 -o gpurun_out/pl_after_libb -f python profiles/run_spmv.py powerlaw8M CSR/LibB 3 > gpurun_out/pl_after_libb.log 2>&1
