#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_mas_apply_l0|k_tet_grad|k_bsr_spmv|k_coarse_mv" -s 40 -c 6 -o gpurun_out/prof_hot4 python tools/c2_iters.py 5e-3 3 30 60 > /dev/null 2>&1
ls gpurun_out
