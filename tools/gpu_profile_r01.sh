#!/bin/bash
# Round-1 profiling pass (run through gpurun): the bench line, the ncu launch
# list of the bench's timed region, and one --set full capture of the
# roofline kernel (k_mas_apply_l0) and of the top CCD / build kernels.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 60000 -c 30000 \
    --log-file gpurun_out/prof/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
for k in "k_mas_apply_l0" "k_tet_grad" "k_bsr_spmv" "k_mas_sweep" "k_block_sweep" "k_hq_edges" "k_pairs_app" "k_tet_hessian" "k_hess_gather"; do
  ncu --set full --import-source on --kernel-name-base demangled -k "regex:^(void )?${k}" --launch-skip 40 --launch-count 1 \
      -o gpurun_out/prof/full_${k} python tools/frames_probe.py 3 60 > gpurun_out/prof/ncu_full_${k}.log 2>&1
done
ls -la gpurun_out/prof
