#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SPMVTUNE_E2E_STEPS=8 timeout 1500 python profiles/e2e_slab_phases.py > gpurun_out/e2e_pool.log 2>&1
echo "rc=$?" >> gpurun_out/e2e_pool.log
