#!/bin/bash
# round 2, call a: GPU test suite, C2 state dump, C3 coarse SPD probe
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gpu_tests.log
timeout 300 python tools/c2_dump.py 5 3 > gpurun_out/r2a_c2_dump.log 2>&1
timeout 1200 python tools/c3_spd_probe.py 1000 2 200 > gpurun_out/r2a_c3_probe.log 2>&1
echo done
