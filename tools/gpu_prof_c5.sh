#!/bin/bash
# config-5 kernel profiles + the reference arm's timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c5_launches.csv python profiles/run_config5_kernels.py --iters 12 > gpurun_out/c5_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_dia|k_dot|k_dcg" -s 20 -c 4 \
    -o gpurun_out/c5_full -f python profiles/run_config5_kernels.py --iters 6 > gpurun_out/c5_full.log 2>&1
( time timeout 2400 python bench.py --impl reference --steps ${STEPS:-5} --warmup ${WARMUP:-3} ) > gpurun_out/ref_arm.log 2>&1
