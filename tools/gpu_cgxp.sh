#!/bin/bash
# CG x/p regrouping: distributed GPU tests, default bench, config-5 launch list; advisor kernel profiles
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_slab_restart.py -q -x > gpurun_out/cg_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/cg_tests.log
timeout 2400 python bench.py --steps ${STEPS:-5} --warmup ${WARMUP:-3} --no-extra > gpurun_out/cg_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/cg_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c5_launches.csv python profiles/run_config5_kernels.py --iters 12 > gpurun_out/c5_launch.log 2>&1
bash tools/gpu_featprof.sh
