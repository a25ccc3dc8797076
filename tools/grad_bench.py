"""GPU micro-benchmark of the SNH gradient kernel on the config-2 scene."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c2_stack(gap=5e-3)
ctx = scene.context(solver.SolverConfig())
x0 = scene.mesh.rest_positions.ravel().copy()
xt = x0 - 1e-4
g0 = ctx.gradient(x0 + 1e-3 * np.sin(np.arange(x0.size)), xt, 0.01)
for _ in range(2):
    ctx.stage_timing(True)
    for _ in range(50):
        g = ctx.gradient(x0 + 1e-3 * np.sin(np.arange(x0.size)), xt, 0.01)
    ms, cnt, b = ctx.stage_stats()["tet_grad"]
    print(f"k_tet_grad<SNH>: {1e3 * ms / cnt:7.2f} us  {b / cnt / (ms / cnt * 1e-3) / 1e9:7.1f} GB/s  "
          f"|g - g0| = {np.abs(g - g0).max():.1e}", flush=True)
