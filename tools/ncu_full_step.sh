#!/bin/bash
# Launch list + one `ncu --set full` capture of every library kernel of one C2 d=64
# truncation step (GPU box).  Reports stay in /tmp; CSV exports go to gpurun_out/.
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py ${STEP_ARGS:-} > gpurun_out/ncu_launches.log 2>&1
cp gpurun_out/tags.json gpurun_out/tags_launches.json
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:_kernel" -f -o /tmp/step_full python tools/profile_step.py ${STEP_ARGS:-} > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/step_full.ncu-rep --page raw --csv > gpurun_out/step_full_raw.csv 2>/dev/null
ncu -i /tmp/step_full.ncu-rep --page details --csv > gpurun_out/step_full_details.csv 2>/dev/null
tail -n 2 gpurun_out/ncu_full.log
