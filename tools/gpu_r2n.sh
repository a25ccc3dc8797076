#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_c2_scale.py tests/test_gpu_parity.py tests/test_gpu_baselines.py -x -q > gpurun_out/r2n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.log
timeout 600 python tools/c5_probe.py > gpurun_out/r2n_c5_probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2n_bench.log 2>&1
timeout 600 python tools/big_scene_run.py c3 2 60 > gpurun_out/r2n_c3.log 2>&1
echo done
