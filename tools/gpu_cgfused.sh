#!/bin/bash
# fused CG iteration: distributed GPU tests, default bench, config-5 launch list + one full capture
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/cg_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/cg_tests.log
timeout 2400 python bench.py --steps ${STEPS:-5} --warmup ${WARMUP:-3} > gpurun_out/cg_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/cg_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c5_launches.csv python profiles/run_config5_kernels.py --iters 12 > gpurun_out/c5_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dia_cg|k_dcg_rupdate" -s 6 -c 2 \
    -o gpurun_out/c5_cg_full -f python profiles/run_config5_kernels.py --iters 6 > gpurun_out/c5_full.log 2>&1
