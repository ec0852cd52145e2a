#!/bin/bash
# full default bench (config 5 at N=1) + the driver's step shape
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/bench_full.log
timeout 2400 python bench.py --steps ${STEPS:-5} --warmup ${WARMUP:-3} >> gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
