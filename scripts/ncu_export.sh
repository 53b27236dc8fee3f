#!/bin/bash
# Summarise an ncu report on the GPU box (the .ncu-rep itself is too large to
# bring back): raw metrics CSV of the kernels + per-kernel source-level stalls.
# usage: scripts/ncu_export.sh <report.ncu-rep> <out_prefix>
rep=$1; out=$2
ncu -i "$rep" --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed > "${out}_raw.csv" 2>&1
python scripts/ncu_top.py "$rep" "" 10 > "${out}_stalls.txt" 2>&1
ncu -i "$rep" --page details --csv > "${out}_details.csv" 2>&1
gzip -f "${out}_details.csv"
