#!/bin/bash
# round 2, call c: where the restart path's time goes with the new coarse kernel
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_coarse_sweep|k_mas_sweep|k_coarse_gather|k_sym_lower|k_coarse_up|k_contact_coarse|k_bsr_to_blocks|k_contact_blocks" -c 60 --csv --log-file gpurun_out/r2c_build_launches.csv python tools/build_bench.py 2 > gpurun_out/r2c_build.log 2>&1
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2c_build_bench.log 2>&1
MP_SERIAL_BUILD=1 timeout 300 python tools/build_bench.py 2 >> gpurun_out/r2c_build_bench.log 2>&1
echo done
