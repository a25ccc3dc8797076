#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_gpu_variants.py tests/test_gpu_baselines.py tests/test_gpu_solver_suite.py tests/test_gpu_multi.py -q > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
timeout 600 python tools/big_scene_run.py c5 1 10 > gpurun_out/r2k_c5.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2k_bench.log 2>&1
echo done
