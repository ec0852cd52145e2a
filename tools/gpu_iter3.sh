#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -k "not config3_cg" > gpurun_out/t3.log 2>&1
echo "tests rc=$?" >> gpurun_out/t3.log
: > gpurun_out/dia5.log
for v in 0 1; do SPMVTUNE_DIA=$v timeout 300 python profiles/bench_dia.py 600 20 >> gpurun_out/dia5.log 2>&1; done
timeout 1200 python bench.py --steps 3 --warmup 1 --no-cpu --no-extra --no-e2e > gpurun_out/bench_c5b.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_c5b.log
