#!/bin/bash
# fp32 + fp64 SpMV sweeps (configs 1-3 matrices) and one full ncu capture of the config-5 DIA SpMV+dot kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SWEEP_DTYPE=f32 timeout 900 python profiles/sweep_spmv.py 30 poisson1024,convdiff2000,powerlaw8M > gpurun_out/sw_f32.json 2> gpurun_out/sw_f32.log
timeout 900 python profiles/sweep_spmv.py 30 poisson1024,convdiff2000,powerlaw8M > gpurun_out/sw_f64.json 2> gpurun_out/sw_f64.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_dia_reg" -s 3 -c 1 \
    -o gpurun_out/c5_dia_full -f python profiles/run_config5_kernels.py --iters 4 > gpurun_out/c5_dia_full.log 2>&1
