#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_slab_restart.py tests/test_gpu_distributed.py tests/test_gpu_solver.py -q -x > gpurun_out/t2.log 2>&1
echo "tests rc=$?" >> gpurun_out/t2.log
: > gpurun_out/dia.log
for v in 0 1; do SPMVTUNE_DIA=$v timeout 300 python profiles/bench_dia.py 600 20 >> gpurun_out/dia.log 2>&1; done
for ns in 2 3; do SPMVTUNE_DIA_NS=$ns timeout 300 python profiles/bench_dia.py 600 20 >> gpurun_out/dia.log 2>&1; done
SPMVTUNE_DIA=0 timeout 300 python profiles/bench_dia.py 300 50 >> gpurun_out/dia.log 2>&1
timeout 300 python profiles/bench_dia.py 300 50 >> gpurun_out/dia.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 1 --no-cpu --no-extra --no-e2e > gpurun_out/bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_c5.log
