#!/bin/bash
# round-end shape: GPU suite, smoke, default bench line, reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/final_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/final_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 2400 python bench.py > gpurun_out/final_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/final_bench.log
( time timeout 2400 python bench.py --impl reference ) > gpurun_out/final_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/final_ref.log
