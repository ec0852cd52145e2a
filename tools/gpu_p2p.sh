#!/bin/bash
# peer-memory collectives: world-2 CUDA path on one GPU (CUDA IPC between two processes)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x -rw > gpurun_out/p2p_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p2p_tests.log
