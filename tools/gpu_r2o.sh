#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2o_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_gpu_tests.log
timeout 600 python tools/c5_probe.py > gpurun_out/r2o_c5_probe.log 2>&1
timeout 600 python tools/big_scene_run.py c5 2 30 > gpurun_out/r2o_c5.log 2>&1
timeout 600 python tools/big_scene_run.py c3 2 60 > gpurun_out/r2o_c3.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2o_bench.log 2>&1
echo done
