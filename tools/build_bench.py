"""GPU micro-benchmark of the restart path on the config-2 scene at a
contact state: H_base assembly and MAS build (CUDA events)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c2_stack(gap=5e-3)
levels = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = solver.SolverConfig(iter_max=200, levels=levels)
ctx = scene.context(cfg)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
if os.path.exists("tools/_data/c2_state_w5.npz"):  # the bench's first timed frame (tools/c2_dump.py)
    x = np.load("tools/_data/c2_state_w5.npz")["x0"]
elif os.path.exists("tools/_data/ccd_state.npz"):
    x = np.load("tools/_data/ccd_state.npz")["x"]
else:
    for _ in range(4):  # reach contact
        ctx.step_device(0.01)
    x, _ = ctx.get_state()
print(f"levels={levels}")
for rep in range(2):
    ctx.stage_timing(True)
    for _ in range(20):
        ctx.snapshot(x, 0.01, build_mas=True)
    st = ctx.stage_stats()
    for k in ("hessian", "mas_build"):
        ms, cnt, b = st[k]
        print(f"{k:10s} {1e3 * ms / cnt:9.1f} us/call" + (f"  {b / cnt / (ms / cnt * 1e-3) / 1e9:7.1f} GB/s" if b else ""),
              flush=True)
