#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2q_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_gpu_tests.log
( time timeout 1200 python bench.py --steps 3 --warmup 5 ) > gpurun_out/r2q_bench.log 2>&1
bash tools/gpu_profile_r02.sh > gpurun_out/r2q_profile.log 2>&1
echo done
