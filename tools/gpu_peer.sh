#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_distributed.py -q -x > gpurun_out/peer_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/peer_tests.log
