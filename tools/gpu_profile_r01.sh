#!/bin/bash
# Round-1 profiling pass (run through gpurun): the bench line, the ncu launch
# list of the bench's timed region (summarised on the box), and --set full
# captures of the roofline kernel and the top kernels (summaries kept; only
# the roofline kernel's report is brought back -- gpurun returns <= 64 MiB).
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 60000 -c 30000 \
    --log-file /tmp/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
python tools/launch_summary.py /tmp/launches_bench.csv 60 > gpurun_out/prof/launches_bench.txt
gzip -c /tmp/launches_bench.csv > gpurun_out/prof/launches_bench.csv.gz
for k in "k_mas_apply_l0_direct" "k_tet_grad" "k_bsr_spmv" "k_mas_sweep" "k_block_sweep" "k_hq_edges" "k_pairs_app" "k_tet_hessian" "k_hess_gather"; do
  ncu --set full --import-source on --kernel-name-base demangled -k "regex:^(void )?${k}[<(]" --launch-skip 40 --launch-count 1 \
      -o /tmp/full_${k} python tools/frames_probe.py 3 60 > /tmp/ncu_full_${k}.log 2>&1
  python tools/ncu_summary.py /tmp/full_${k}.ncu-rep > gpurun_out/prof/full_${k}.txt 2>&1
  ncu -i /tmp/full_${k}.ncu-rep --page raw --csv > /tmp/raw_${k}.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/raw_${k}.csv >> gpurun_out/prof/full_${k}.txt 2>&1
done
cp /tmp/full_k_mas_apply_l0_direct.ncu-rep gpurun_out/prof/ 2>/dev/null
du -sh gpurun_out/prof; ls -la gpurun_out/prof
