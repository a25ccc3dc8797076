#!/bin/bash
# round 2, call b: cuBLAS-free coarse inverse -- unit tests, parity suite, C3 probe, restart-path timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_variants.py -x -q > gpurun_out/r2b_coarse_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_coarse_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_gpu_tests.log
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2b_build_bench.log 2>&1
OUT=gpurun_out/r2b timeout 1500 python tools/c3_spd_probe.py 1000 2 200 > gpurun_out/r2b_c3_probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2b_bench.log 2>&1
echo done
