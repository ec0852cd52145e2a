#!/bin/bash
# a larger B200 training corpus for the cascade (630 generated matrices, seed 2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ds2
( time timeout 3300 python -m paper_2411_10143_b200 dataset --generated 630 --seed 2 --out gpurun_out/ds2 ) > gpurun_out/ds2.log 2>&1
echo "rc=$?" >> gpurun_out/ds2.log
