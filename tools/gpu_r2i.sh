#!/bin/bash
# round 2, call i: checker + CLI on the GPU, coarse kernel, big scenes (C3/C4/C5) sizing runs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_gpu_coarse.py tests/test_gpu_c2_scale.py -x -q > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
timeout 300 python tools/build_bench.py 2 > gpurun_out/r2i_build_bench.log 2>&1
timeout 900 python tools/big_scene_run.py c5 2 60 > gpurun_out/r2i_c5.log 2>&1
timeout 900 python tools/big_scene_run.py c4 2 60 > gpurun_out/r2i_c4.log 2>&1
timeout 900 python tools/big_scene_run.py c3 2 60 > gpurun_out/r2i_c3.log 2>&1
echo done
