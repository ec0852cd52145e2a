#!/bin/bash
# config-3 (power-law 8M) SpMV: launch list + one full ncu capture per row kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TOKS=${TOKS:-CSR/LibB,CSR/LibA/32,HYB/LibA,COO/LibB}
TAG=${TAG:-pl8}
timeout 600 python profiles/sweep_spmv.py 20 powerlaw8M > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python profiles/run_spmv.py powerlaw8M $TOKS 3 > gpurun_out/${TAG}_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_rows_pipe|k_ell|k_coo" -s 2 -c 8 \
    -o gpurun_out/${TAG}_full -f python profiles/run_spmv.py powerlaw8M $TOKS 3 > gpurun_out/${TAG}_full.log 2>&1
echo done >> gpurun_out/${TAG}_full.log
