#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_gpu_tests.log
timeout 600 python tools/c5_frame1.py 20 > gpurun_out/r2s_c5_frame1.log 2>&1
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2s_build_bench.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 5 --configs c3,c5 > gpurun_out/r2s_bench.log 2>&1
echo done
