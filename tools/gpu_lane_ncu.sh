#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__shared_mem_per_block_dynamic,dram__bytes_read.sum,lts__t_sector_hit_rate.pct
SPMVTUNE_LIB_VARIANT=old timeout 300 ncu --metrics $M --clock-control none --csv -k regex:k_rows_pipe --log-file gpurun_out/lane_old.csv python profiles/run_spmv.py convdiff2000 CSR/LibA/2 3 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv -k regex:k_rows_pipe --log-file gpurun_out/lane_new.csv python profiles/run_spmv.py convdiff2000 CSR/LibA/2 3 > /dev/null 2>&1
