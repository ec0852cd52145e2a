#!/bin/bash
# N=2 bench flow on ONE GPU (gloo-staged base comm; peer-memory layer on/off) at 200^3 — path validation, not a number
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export SPMVTUNE_DIST_BACKEND=gloo SPMVTUNE_CONFIG5_N=200
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --no-extra > gpurun_out/n2_p2p.log 2>&1
echo "rc=$?" >> gpurun_out/n2_p2p.log
SPMVTUNE_P2P=0 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --no-extra > gpurun_out/n2_base.log 2>&1
echo "rc=$?" >> gpurun_out/n2_base.log
timeout 600 python bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu --no-extra > gpurun_out/n1_200.log 2>&1
echo "rc=$?" >> gpurun_out/n1_200.log
