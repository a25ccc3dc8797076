#!/bin/bash
# Closing round-2 profiling pass (through gpurun): the launch list of one
# bench frame and --set full captures of the kernels changed late in the
# round (flattened grid queries, MAS build, BVH).  Summaries only come back.
mkdir -p gpurun_out/prof3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_frame.csv \
    python tools/frame_profile.py 500 > gpurun_out/prof3/frame_profile.log 2>&1
python tools/launch_summary.py /tmp/launches_frame.csv 60 > gpurun_out/prof3/launches_frame.txt
gzip -c /tmp/launches_frame.csv > gpurun_out/prof3/launches_frame.csv.gz
for k in "k_mas_apply_l0_direct" "k_hq_edges" "k_mas_sweep" "k_coarse_sweep" "k_contact_coarse" "k_coarse_gather"; do
  timeout 600 ncu --set full --import-source on --kernel-name-base demangled -k "regex:^(void )?${k}[<(]" --launch-skip 6 --launch-count 1 \
      -o /tmp/full_${k} python tools/frame_profile.py 20 > /tmp/ncu_full_${k}.log 2>&1
  python tools/ncu_summary.py /tmp/full_${k}.ncu-rep > gpurun_out/prof3/full_${k}.txt 2>&1
  ncu -i /tmp/full_${k}.ncu-rep --page raw --csv > /tmp/raw_${k}.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/raw_${k}.csv >> gpurun_out/prof3/full_${k}.txt 2>&1
done
du -sh gpurun_out/prof3; ls gpurun_out/prof3
