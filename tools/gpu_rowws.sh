#!/bin/bash
# warp-specialised row kernel: exactness (forced on every matrix), sweep ws vs cta and tile variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SPMVTUNE_ROWKERNEL=ws timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_scale.py tests/test_gpu_edge_cases.py -q -x -k "not config3_cg and not tma_arnoldi and not fallback" > gpurun_out/ws_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ws_tests.log
: > gpurun_out/ws_sweep.log
for c in 0 6 7 8; do
  echo "ws cfg=$c" >> gpurun_out/ws_sweep.log
  SPMVTUNE_ROWCFG=$c SPMVTUNE_ROWKERNEL=ws SWEEP_TOKENS=CSR/LibB,CSR/LibA/32,CSR/LibA/8,COO/LibA,HYB/LibA timeout 600 python profiles/sweep_spmv.py 20 ${MATS:-powerlaw8M} 2>> gpurun_out/ws_sweep.log >/dev/null
done
echo "ws default on stencils" >> gpurun_out/ws_sweep.log
SPMVTUNE_ROWKERNEL=ws SWEEP_TOKENS=CSR/LibB,CSR/LibA/32,COO/LibA timeout 600 python profiles/sweep_spmv.py 20 poisson1024,convdiff2000 2>> gpurun_out/ws_sweep.log >/dev/null
ncu --set full --import-source on --clock-control none -k regex:"k_rows_ws" -s 1 -c 2 \
    -o gpurun_out/ws_full -f python profiles/run_spmv.py powerlaw8M CSR/LibB,CSR/LibA/32 3 > gpurun_out/ws_full.log 2>&1
