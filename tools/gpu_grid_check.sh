#!/bin/bash
# GPU tests, the Arnoldi grid A/B with the automatic rule, config-4 suite (native loop)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/gc
(timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8) > gpurun_out/gc/tests.log
cat gpurun_out/gc/tests.log
SPMVTUNE_MGS_GRID=0 timeout 300 python profiles/mgs_grid_ab.py 0 > gpurun_out/gc/auto.txt 2>&1
tail -n 1 gpurun_out/gc/auto.txt | cut -c1-600
for ms in tests/golden/models paper_2411_10143_b200/models/b200; do
  tag=$(basename $ms)
  timeout 900 python -m paper_2411_10143_b200 suite --models $ms --out gpurun_out/gc/suite_$tag > gpurun_out/gc/suite_$tag.log 2>&1
  python -m paper_2411_10143_b200 report gpurun_out/gc/suite_$tag --out gpurun_out/gc/suite_$tag.csv > gpurun_out/gc/suite_$tag.txt 2>&1
  tail -n 2 gpurun_out/gc/suite_$tag.txt
done
