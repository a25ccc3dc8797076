#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_c2_scale.py -x -q > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 900 python tools/big_scene_run.py c5 2 60 > gpurun_out/r2j_c5.log 2>&1
timeout 900 python tools/big_scene_run.py c4 2 60 > gpurun_out/r2j_c4.log 2>&1
timeout 900 python tools/big_scene_run.py c3 2 60 > gpurun_out/r2j_c3.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2j_bench.log 2>&1
echo done
