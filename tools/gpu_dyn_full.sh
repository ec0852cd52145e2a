#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/dynf_tests.log 2>&1
echo "rc=$?" >> gpurun_out/dynf_tests.log
timeout 900 python profiles/config_details.py config3 config1 > gpurun_out/dynf_details.log 2>&1
