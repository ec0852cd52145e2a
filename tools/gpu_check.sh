#!/bin/bash
# full GPU suite + smoke + default bench line (the driver's round-end shape)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/check_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/check_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/check_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/check_smoke.log
timeout 2400 python bench.py --steps ${STEPS:-5} --warmup ${WARMUP:-3} > gpurun_out/check_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/check_bench.log
