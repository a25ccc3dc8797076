#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_baselines.py -q > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
timeout 420 python tools/big_scene_run.py c5 1 10 > gpurun_out/r2l_c5.log 2>&1
timeout 600 python tools/big_scene_run.py c3 2 60 > gpurun_out/r2l_c3.log 2>&1
echo done
