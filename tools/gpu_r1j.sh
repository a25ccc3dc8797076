#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
# launch list inside the first timed frame (skips the 3 warm-up frames' launches)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 45000 -c 25000 --csv --log-file gpurun_out/launches_bench_timed.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_mas_apply_l0|k_tet_grad|k_bsr_spmv|k_mas_sweep|k_block_sweep|k_pairs|k_hq_edges" -s 200 -c 8 -o gpurun_out/prof_r01 python tools/c2_iters.py 5e-3 4 40 60 > /dev/null 2>&1
ls gpurun_out
