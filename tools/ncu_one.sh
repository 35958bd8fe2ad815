#!/bin/bash
# One `ncu --set full` capture (with source) of the first launch of kernel regex $1
# inside one C2 step; raw + source-page CSVs to gpurun_out/<tag>_*.csv.
#   bash tools/ncu_one.sh 'gemm_kernel' tag [skip]
set -u
mkdir -p gpurun_out
K="$1"; TAG="$2"; SKIP="${3:-0}"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:$K" -s "$SKIP" -c 1 -f -o /tmp/$TAG python tools/profile_step.py > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
cp /tmp/$TAG.ncu-rep gpurun_out/ 2>/dev/null
tail -n 3 gpurun_out/${TAG}_ncu.log
