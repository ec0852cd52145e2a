#!/bin/bash
# A/B of the row kernel: previous build (libspmvtune_b200_old.so) vs current, same box, alternating
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
SPMVTUNE_LIB_VARIANT=old timeout 600 python profiles/sweep_spmv.py 40 poisson1024,convdiff2000,powerlaw8M > gpurun_out/ab_old_$r.json 2>/dev/null
timeout 600 python profiles/sweep_spmv.py 40 poisson1024,convdiff2000,powerlaw8M > gpurun_out/ab_new_$r.json 2>/dev/null
done
timeout 1200 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_scale.py tests/test_gpu_solver.py -q -x > gpurun_out/ab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/ab_tests.log
