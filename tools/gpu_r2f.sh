#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/frame_profile.py > gpurun_out/r2f_frame_profile.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches_frame.csv python tools/frame_profile.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2f_launches_frame.csv > gpurun_out/r2f_launches_frame.txt 2>&1
gzip -f gpurun_out/r2f_launches_frame.csv
MP_CS_PROF=1 timeout 300 python tools/coarse_prof.py 276 1095 > gpurun_out/r2e_coarse_prof.log 2>&1
echo done
