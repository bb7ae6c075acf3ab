#!/bin/bash
# Executed instructions per element of every map kernel (one ncu metrics pass):
# bash tools/gpu_inst.sh TAG [perf.py args]  -> gpurun_out/inst_TAG.csv + table
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:'k_map_vec|k_sincos_vec|k_f64' --csv --log-file gpurun_out/inst_$TAG.csv \
  python tools/perf.py --reps 1 "$@" > /dev/null 2>&1
python tools/inst_table.py gpurun_out/inst_$TAG.csv
