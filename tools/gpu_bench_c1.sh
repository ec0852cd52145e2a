#!/bin/bash
# full default bench line, then the config-1 A/B driver in a fresh process
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2000 python bench.py > gpurun_out/bc1_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bc1_bench.log
timeout 600 python profiles/c1_ab.py > gpurun_out/bc1_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/bc1_ab.log
