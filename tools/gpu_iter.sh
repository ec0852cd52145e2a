#!/bin/bash
# one GPU iteration: new GPU tests + a small bench run (paths validation)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slab_restart.py tests/test_gpu_scale.py tests/test_gpu_spmv.py -q -x -k "not config3" > gpurun_out/t_new.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_new.log
SPMVTUNE_CONFIG5_N=200 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_small.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_small.log
