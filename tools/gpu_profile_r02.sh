#!/bin/bash
# Round-2 profiling pass (through gpurun): the launch list of one bench frame
# (frame 6 from the committed start state), --set full captures of the top
# kernels inside a 20-iteration frame, and FP64-pipe utilisation of the
# compute-bound build kernels.  Summaries only come back (<= 64 MiB).
mkdir -p gpurun_out/prof2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_frame.csv \
    python tools/frame_profile.py 500 > gpurun_out/prof2/frame_profile.log 2>&1
python tools/launch_summary.py /tmp/launches_frame.csv 60 > gpurun_out/prof2/launches_frame.txt
gzip -c /tmp/launches_frame.csv > gpurun_out/prof2/launches_frame.csv.gz
for k in "k_mas_apply_l0_direct" "k_coarse_sweep" "k_mas_sweep" "k_tet_grad" "k_grad_gather" "k_hq_edges" "k_pairs_app" "k_tet_hessian" "k_hess_gather" "k_bsr_spmv"; do
  timeout 600 ncu --set full --import-source on --kernel-name-base demangled -k "regex:^(void )?${k}[<(]" --launch-skip 6 --launch-count 1 \
      -o /tmp/full_${k} python tools/frame_profile.py 20 > /tmp/ncu_full_${k}.log 2>&1
  python tools/ncu_summary.py /tmp/full_${k}.ncu-rep > gpurun_out/prof2/full_${k}.txt 2>&1
  ncu -i /tmp/full_${k}.ncu-rep --page raw --csv > /tmp/raw_${k}.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/raw_${k}.csv >> gpurun_out/prof2/full_${k}.txt 2>&1
  grep -o '"[^"]*pipe_fp64[^"]*","[^"]*","[^"]*"' /tmp/raw_${k}.csv | head -4 >> gpurun_out/prof2/full_${k}.txt
done
cp /tmp/full_k_mas_apply_l0_direct.ncu-rep /tmp/full_k_coarse_sweep.ncu-rep gpurun_out/prof2/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k "regex:k_coarse_sweep|k_mas_sweep|k_tet_hessian" -c 12 --csv --log-file gpurun_out/prof2/fp64_pipe.csv \
    python tools/build_bench.py 2 > /dev/null 2>&1
du -sh gpurun_out/prof2; ls gpurun_out/prof2
