#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -12 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python tools/bp_probe.py > gpurun_out/bp_probe.txt 2>&1
cat gpurun_out/bp_probe.txt
timeout 400 python tools/c2_probe.py 2 100 > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
