#!/bin/bash
# round 2, call d: fused level-0 build + faster coarse kernel; C2-scale parity vs the reference
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_gpu_tests.log
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2d_build_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_coarse_sweep|k_mas_sweep|k_coarse_gather|k_sym_lower|k_coarse_up|k_contact_coarse|k_tet_hessian|k_hess_gather|k_fx_scale" -c 40 --csv --log-file gpurun_out/r2d_build_launches.csv python tools/build_bench.py 2 > /dev/null 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench.log 2>&1
echo done
