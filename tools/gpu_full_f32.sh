#!/bin/bash
# whole GPU suite (incl. the config-5 family at 120^3) + fp32 sweep after the multi-row fp32 DIA kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/full_tests.log
SWEEP_DTYPE=f32 timeout 900 python profiles/sweep_spmv.py 30 poisson1024,convdiff2000 > gpurun_out/sw_f32b.json 2> gpurun_out/sw_f32b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1
