#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -12 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python tools/c2_iters.py 5e-3 8 40 200 > gpurun_out/c2_iters.txt 2>&1
grep frame gpurun_out/c2_iters.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 6000 --csv --log-file gpurun_out/launches_c2.csv python tools/c2_iters.py 5e-3 4 40 120 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_mas_sweep -s 2 -c 1 -o gpurun_out/prof_sweep python tools/c2_iters.py 5e-3 2 10 60 > /dev/null 2>&1
ls -la gpurun_out/
