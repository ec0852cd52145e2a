#!/bin/bash
# config 4 A/B: the generated 50-matrix suite on the Python solver loop vs the
# native (C++) loop, both model sets (default / sequential / async)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/loop
for loop in python native; do
  for ms in tests/golden/models paper_2411_10143_b200/models/b200; do
    tag=${loop}_$(basename $ms)
    SPMVTUNE_LOOP=$loop timeout 900 python -m paper_2411_10143_b200 suite --models $ms --out gpurun_out/loop/suite_$tag > gpurun_out/loop/suite_$tag.log 2>&1
    python -m paper_2411_10143_b200 report gpurun_out/loop/suite_$tag --out gpurun_out/loop/suite_$tag.csv > gpurun_out/loop/suite_$tag.txt 2>&1
    tail -n 2 gpurun_out/loop/suite_$tag.txt
  done
done
