#!/bin/bash
# config 4: the generated 50-matrix suite, shipped models and the retrained B200 models (default / sequential / async)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for ms in tests/golden/models paper_2411_10143_b200/models/b200; do
  tag=$(basename $ms)
  timeout 1500 python -m paper_2411_10143_b200 suite --models $ms --out gpurun_out/suite_$tag > gpurun_out/suite_$tag.log 2>&1
  python -m paper_2411_10143_b200 report gpurun_out/suite_$tag --out gpurun_out/suite_$tag.csv > gpurun_out/suite_$tag.txt 2>&1
done
