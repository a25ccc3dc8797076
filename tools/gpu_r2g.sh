#!/bin/bash
# round 2, call g: partitioned multi-GPU group (2/3 shards on one GPU) == single GPU; full GPU suite; bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2g_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_multi.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_bench.log 2>&1
echo done
