#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/c5_check_rest.py > gpurun_out/r2m_c5_rest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_c2_scale.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_multi.py -x -q > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2m_c3_launches.csv python tools/big_scene_run.py c3 1 12 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2m_c3_launches.csv > gpurun_out/r2m_c3_launches.txt 2>&1; gzip -f gpurun_out/r2m_c3_launches.csv
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/r2m_bench.log 2>&1
echo done
