#!/bin/bash
# A/B: config-5 bench with the DIA SpMV+dot kernel at 6 CTAs/SM (36 regs) vs 8 CTAs/SM (launch bounds, 31 regs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "" lb8 "" lb8; do
  SPMVTUNE_LIB_VARIANT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/ab_dia_${v:-base}_$RANDOM.log 2>&1
done
