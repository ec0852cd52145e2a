#!/bin/bash
# config 4: advisor stream priority A/B (B200 models, native loop)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/prio
for pr in 1 0 -1; do
  SPMVTUNE_ADVISOR_PRIORITY=$pr timeout 900 python -m paper_2411_10143_b200 suite --models paper_2411_10143_b200/models/b200 --out gpurun_out/prio/suite_$pr > gpurun_out/prio/suite_$pr.log 2>&1
  python -m paper_2411_10143_b200 report gpurun_out/prio/suite_$pr --out gpurun_out/prio/suite_$pr.csv > gpurun_out/prio/suite_$pr.txt 2>&1
  echo "prio $pr"; tail -n 2 gpurun_out/prio/suite_$pr.txt
done
