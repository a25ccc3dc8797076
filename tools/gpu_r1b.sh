#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python tools/c2_probe.py 3 200 > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
