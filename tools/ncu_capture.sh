#!/bin/bash
# ncu captures of one C2 d=64 truncation step (run on the GPU box via gpurun).
# Big .ncu-rep files stay in /tmp; CSV exports land in gpurun_out/.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py > $OUT/ncu_launches.log 2>&1
cap() {  # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k "regex:$2" --launch-skip $3 --launch-count $4 -f -o /tmp/$1 python tools/profile_step.py > $OUT/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > $OUT/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
  sz=$(stat -c %s /tmp/$1.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 12000000 ]; then cp /tmp/$1.ncu-rep $OUT/; fi
}
for spec in "$@"; do
  cap $spec
done
