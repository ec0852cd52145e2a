#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/dia4.log
for v in 0 7 8 9 10 11 12; do SPMVTUNE_DIA=$v timeout 300 python profiles/bench_dia.py 600 20 >> gpurun_out/dia4.log 2>&1; done
for v in 0 7 9 10; do SPMVTUNE_DIA=$v timeout 300 python profiles/bench_dia.py 300 50 >> gpurun_out/dia4.log 2>&1; done
