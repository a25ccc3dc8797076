#!/bin/bash
# round 2, call h: coarse-inverse lookahead -- unit tests, timing, C2 parity, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_c2_scale.py tests/test_gpu_multi.py -x -q > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
MP_CS_PROF=1 timeout 300 python tools/coarse_prof.py 276 1095 1902 > gpurun_out/r2h_coarse_prof.log 2>&1
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2h_build_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_coarse_sweep|k_mas_sweep" -c 12 --csv --log-file gpurun_out/r2h_build_launches.csv python tools/build_bench.py 2 > /dev/null 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench.log 2>&1
echo done
